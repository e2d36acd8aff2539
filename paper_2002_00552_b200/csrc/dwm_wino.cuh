// dwm_wino.cuh -- compile-time Winograd F(2, r<=3) coefficients and exact
// sequential-sum helpers shared by the fused small-C kernel and the input
// transform.  Coefficients are 0 / +-1 (Bt, At); zero terms are skipped and
// +-1 terms are exact adds/subs in ascending index order, which reproduces the
// reference's BLAS contraction (engines.py:71-79) bit for bit up to the sign
// of exact zeros.
#pragma once
#include <utility>

namespace dwm {
namespace wino {

// At coefficient of F(2, r): row i (output), column a (frequency).
__host__ __device__ constexpr int at_coef(int r, int i, int a) {
  return r == 1 ? (i == a ? 1 : 0)
       : r == 2 ? (i == 0 ? (a <= 1 ? 1 : 0) : (a == 1 ? 1 : (a == 2 ? -1 : 0)))
                : (i == 0 ? (a <= 2 ? 1 : 0) : (a == 0 ? 0 : (a == 1 ? 1 : -1)));
}
// Bt coefficient of F(2, r): row a (frequency), column i (window sample).
__host__ __device__ constexpr int bt_coef(int r, int a, int i) {
  // F(2,1): I2;  F(2,2): [[1,-1,0],[0,1,0],[0,1,-1]];
  // F(2,3): [[1,0,-1,0],[0,1,1,0],[0,-1,1,0],[0,1,0,-1]]
  return r == 1 ? (a == i ? 1 : 0)
       : r == 2 ? (a == 0 ? (i == 0 ? 1 : i == 1 ? -1 : 0)
                  : a == 1 ? (i == 1 ? 1 : 0)
                           : (i == 1 ? 1 : i == 2 ? -1 : 0))
                : (a == 0 ? (i == 0 ? 1 : i == 2 ? -1 : 0)
                  : a == 1 ? (i == 1 || i == 2 ? 1 : 0)
                  : a == 2 ? (i == 1 ? -1 : i == 2 ? 1 : 0)
                           : (i == 1 ? 1 : i == 3 ? -1 : 0));
}
// first index with a nonzero coefficient (the sequential sum starts there)
__host__ __device__ constexpr int at_first(int r, int i) {
  int k = 0;
  while (at_coef(r, i, k) == 0) ++k;
  return k;
}
__host__ __device__ constexpr int bt_first(int r, int a) {
  int k = 0;
  while (bt_coef(r, a, k) == 0) ++k;
  return k;
}

// ---- scalar chain (producer): acc = sum_k K_k * m_k, K in {0, +-1} ---------
// Zero terms are skipped and the first nonzero term is a move (BLAS starts from
// +0, so only the sign of an exact zero can differ).  A leading -1 (Bt row 2
// of F(2,3)) is carried as a negated accumulator and fixed by `finish`.
__device__ __forceinline__ float wadd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double wadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float wsub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double wsub(double a, double b) { return __dsub_rn(a, b); }
template <int K, bool FIRST, bool NEG, typename T> __device__ __forceinline__ void chain(T& acc, T m) {
  if constexpr (K == 0) return;
  else if constexpr (FIRST) acc = m;  // value is K*m; sign kept in NEG
  else if constexpr ((K == 1) != NEG) acc = wadd(acc, m);
  else acc = wsub(acc, m);
}

template <typename F, int... Is>
__device__ __forceinline__ void static_for_impl(F&& f, std::integer_sequence<int, Is...>) {
  (f(std::integral_constant<int, Is>{}), ...);
}
template <int N, typename F> __device__ __forceinline__ void static_for(F&& f) {
  static_for_impl(f, std::make_integer_sequence<int, N>{});
}


// Bt.d.B of one part window (row stage then column stage) with compile-time
// coefficients; calls store(q, value) for q = a*(PC+1) + b.
template <int PR, int PC, typename T, typename Store>
__device__ __forceinline__ void input_transform_part(const T (&win)[4][4], Store&& store) {
  constexpr int LR = PR + 1, LC = PC + 1;
  T tt[LR][LC];
  static_for<LR>([&](auto aI) {
    constexpr int a = decltype(aI)::value;
    constexpr bool neg = bt_coef(PR, a, bt_first(PR, a)) < 0;
    static_for<LR>([&](auto iI) {
      constexpr int i = decltype(iI)::value;
#pragma unroll
      for (int j = 0; j < LC; ++j) chain<bt_coef(PR, a, i), (i == bt_first(PR, a)), neg>(tt[a][j], win[i][j]);
    });
    if constexpr (neg) {
#pragma unroll
      for (int j = 0; j < LC; ++j) tt[a][j] = -tt[a][j];
    }
  });
  static_for<LR>([&](auto aI) {
    constexpr int a = decltype(aI)::value;
    static_for<LC>([&](auto bI) {
      constexpr int b = decltype(bI)::value;
      constexpr bool neg = bt_coef(PC, b, bt_first(PC, b)) < 0;
      T v;
      static_for<LC>([&](auto jI) {
        constexpr int j = decltype(jI)::value;
        chain<bt_coef(PC, b, j), (j == bt_first(PC, b)), neg>(v, tt[a][j]);
      });
      store(a * LC + b, neg ? -v : v);
    });
  });
}

#define DWM_PART_SWITCH(pr, pc, CALL)            \
  switch ((pr) * 4 + (pc)) {                     \
    case 5: CALL(1, 1); break;                   \
    case 6: CALL(1, 2); break;                   \
    case 7: CALL(1, 3); break;                   \
    case 9: CALL(2, 1); break;                   \
    case 10: CALL(2, 2); break;                  \
    case 11: CALL(2, 3); break;                  \
    case 13: CALL(3, 1); break;                  \
    case 14: CALL(3, 2); break;                  \
    default: CALL(3, 3); break;                  \
  }

}  // namespace wino
}  // namespace dwm
