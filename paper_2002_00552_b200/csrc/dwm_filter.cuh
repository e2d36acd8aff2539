// dwm_filter.cuh -- the per-part filter transform U = G g Gt of one (f, c)
// (reference rows W and U: engines.py:246-248, 187), shared by
// the plain filter transform and the tcgen05 engine's fp16-split variant.
#pragma once
#include "dwm_common.cuh"

namespace dwm {

// Element strides of the weight view the filter transforms read: (f, c, kh, kw).
// The forward passes the contiguous F,C,r_h,r_w layout; the backward's data
// gradient passes the channel-transposed, tap-reversed polyphase sub-kernels
// w[:, :, rho::s_h, sig::s_w] (negative tap strides) without materialising them.
struct FiltView {
  int64_t sf, sc, skh, skw;
};
__host__ __device__ inline FiltView contiguous_view(const dwm_desc_t& d) {
  return FiltView{(int64_t)d.c * d.r_h * d.r_w, (int64_t)d.r_h * d.r_w, d.r_w, 1};
}

template <typename T>
__device__ __forceinline__ void part_filter_transform(const dwm_desc_t& d, const T* __restrict__ wfc, const FiltView& fv,
                                                      int rp, int cp, T out[4][4]) {
  const dwm_axis_part_t R = d.row_parts[rp], Cc = d.col_parts[cp];
  const int pr = R.count, pc = Cc.count;
  T g[3][3];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      g[i][j] = (i < pr && j < pc)
                    ? wfc[(int64_t)(R.origin + R.step * i) * fv.skh + (int64_t)(Cc.origin + Cc.step * j) * fv.skw]
                    : T(0);
  // row stage: t[u][j] = sum_i G_r[u][i] * g[i][j]
  T t[4][3];
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      T acc = mul_rn((T)c_g[pr][u][0], g[0][j]);
#pragma unroll
      for (int i = 1; i < 3; ++i)
        if (i < pr) acc = fma_rn((T)c_g[pr][u][i], g[i][j], acc);
      t[u][j] = acc;
    }
  // column stage: U[u][v] = sum_j t[u][j] * G_c[v][j]
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      T acc = mul_rn(t[u][0], (T)c_g[pc][v][0]);
#pragma unroll
      for (int j = 1; j < 3; ++j)
        if (j < pc) acc = fma_rn(t[u][j], (T)c_g[pc][v][j], acc);
      out[u][v] = acc;
    }
}

}  // namespace dwm
