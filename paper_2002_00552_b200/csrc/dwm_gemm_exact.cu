// dwm_gemm_exact.cu -- transform-domain contraction + fused output transform
// on the CUDA cores, in the reference's exact stage order.
//
// Reference rows: M (engines.py:82-89,189), A (engines.py:192-194),
// Sigma (tensor.py:68-81 at engines.py:254), F (tensor.py:27-30 at engines.py:255).
//
// For every (tile, filter) pair a thread owns, and for every part in plan
// order, frequency by frequency (column frequency b outer, row frequency a
// inner):
//   M      = sum_c U[fq][f][c] * V[fq][tile][c]   FMA chain, c ascending
//   S[i]  += At_r[i][a] * M                       row stage of At.m.A, a ascending
//   T[i][j] += S[i] * At_c[j][b]                  column stage, b ascending
//   y      = y + T                                left fold over parts
// which is the reference's rounding sequence when its BLAS accumulates
// sequentially (small C).  Only y reaches HBM: the per-part outputs and the
// per-frequency products stay in registers; non-finite outputs raise a flag.
#include <cstring>

#include "dwm_common.cuh"
#include "dwm_kernels.h"

namespace dwm {

template <typename T, int BM, int BN, int TM, int TN, int KC>
__global__ void __launch_bounds__((BM / TM) * (BN / TN))
gemm_exact_kernel(const dwm_desc_t d, const T* __restrict__ V, const T* __restrict__ U,
                  T* __restrict__ y, int32_t* __restrict__ flag) {
  constexpr int GM = BM / TM;  // threads along tiles (fast index)
  constexpr int GN = BN / TN;
  constexpr int NT = GM * GN;
  constexpr int VW = 16 / sizeof(T);  // elements per 16-byte vector
  static_assert(TM % VW == 0 || VW % TM == 0, "register tile vs vector width");
  // thread (tm, tn) owns tiles tm*TM .. +TM-1 and filters tn*TN .. +TN-1:
  // contiguous in smem, so the K loop reads them with 16-byte loads
  __shared__ __align__(16) T sV[KC][BM];
  __shared__ __align__(16) T sU[KC][BN];

  const int tid = threadIdx.x;
  const int tm = tid % GM, tn = tid / GM;
  const int64_t tile0 = (int64_t)blockIdx.x * BM;
  const int f0 = blockIdx.y * BN;
  const int C = d.c, F = d.f;
  const int64_t tiles = d.tiles;
  const bool vec = (C % VW) == 0;

  T acc[TM][TN][2][2];
  T Tt[TM][TN][2][2];
  T S[TM][TN][2];

  int fq_base = 0;
  for (int p = 0; p < d.n_row_parts * d.n_col_parts; ++p) {
    const int pr = d.row_parts[p / d.n_col_parts].count;
    const int pc = d.col_parts[p % d.n_col_parts].count;
    const int lr = pr + 1, lc = pc + 1;
    for (int b = 0; b < lc; ++b) {
      for (int a = 0; a < lr; ++a) {
        const int fq = fq_base + a * lc + b;
        const T* Vq = V + (int64_t)fq * tiles * C;
        const T* Uq = U + (int64_t)fq * F * C;
        T M[TM][TN];
        for (int k0 = 0; k0 < C; k0 += KC) {
          const int kn = min(KC, C - k0);
          __syncthreads();
          if (vec) {
            // 16-byte loads along channels, transposed into [k][tile] / [k][filter]
            for (int e = tid; e < BM * (KC / VW); e += NT) {
              const int kq = e % (KC / VW), t = e / (KC / VW);
              const int64_t tile = tile0 + t;
              T v[VW];
              if (tile < tiles && k0 + kq * VW < C) {
                const float4 q = __ldg(reinterpret_cast<const float4*>(Vq + tile * C + k0 + kq * VW));
                memcpy(v, &q, 16);
              } else {
#pragma unroll
                for (int z = 0; z < VW; ++z) v[z] = T(0);
              }
#pragma unroll
              for (int z = 0; z < VW; ++z) sV[kq * VW + z][t] = v[z];
            }
            for (int e = tid; e < BN * (KC / VW); e += NT) {
              const int kq = e % (KC / VW), fl = e / (KC / VW);
              T u[VW];
              if (f0 + fl < F && k0 + kq * VW < C) {
                const float4 q = __ldg(reinterpret_cast<const float4*>(Uq + (int64_t)(f0 + fl) * C + k0 + kq * VW));
                memcpy(u, &q, 16);
              } else {
#pragma unroll
                for (int z = 0; z < VW; ++z) u[z] = T(0);
              }
#pragma unroll
              for (int z = 0; z < VW; ++z) sU[kq * VW + z][fl] = u[z];
            }
          } else {
            for (int e = tid; e < BM * KC; e += NT) {
              const int k = e % KC, t = e / KC;
              const int64_t tile = tile0 + t;
              sV[k][t] = (k < kn && tile < tiles) ? Vq[tile * C + k0 + k] : T(0);
            }
            for (int e = tid; e < BN * KC; e += NT) {
              const int k = e % KC, fl = e / KC;
              sU[k][fl] = (k < kn && f0 + fl < F) ? Uq[(int64_t)(f0 + fl) * C + k0 + k] : T(0);
            }
          }
          __syncthreads();
          for (int k = 0; k < kn; ++k) {
            T vv[TM], uu[TN];
#pragma unroll
            for (int i = 0; i < TM; i += (TM < VW ? TM : VW)) {
              if constexpr (TM * sizeof(T) >= 16) {
                const float4 q = *reinterpret_cast<const float4*>(&sV[k][tm * TM + i]);
                memcpy(vv + i, &q, 16);
              } else {
#pragma unroll
                for (int z = 0; z < TM; ++z) vv[z] = sV[k][tm * TM + z];
              }
            }
#pragma unroll
            for (int j = 0; j < TN; j += (TN < VW ? TN : VW)) {
              if constexpr (TN * sizeof(T) >= 16) {
                const float4 q = *reinterpret_cast<const float4*>(&sU[k][tn * TN + j]);
                memcpy(uu + j, &q, 16);
              } else {
#pragma unroll
                for (int z = 0; z < TN; ++z) uu[z] = sU[k][tn * TN + z];
              }
            }
            if (k0 + k == 0) {
#pragma unroll
              for (int i = 0; i < TM; ++i)
#pragma unroll
                for (int j = 0; j < TN; ++j) M[i][j] = mul_rn(uu[j], vv[i]);
            } else {
#pragma unroll
              for (int i = 0; i < TM; ++i)
#pragma unroll
                for (int j = 0; j < TN; ++j) M[i][j] = fma_rn(uu[j], vv[i], M[i][j]);
            }
          }
        }
        // row stage of At.m.A
        const T ar0 = (T)c_at[pr][0][a], ar1 = (T)c_at[pr][1][a];
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int j = 0; j < TN; ++j) {
            if (a == 0) {
              S[i][j][0] = mul_rn(ar0, M[i][j]);
              S[i][j][1] = mul_rn(ar1, M[i][j]);
            } else {
              S[i][j][0] = fma_rn(ar0, M[i][j], S[i][j][0]);
              S[i][j][1] = fma_rn(ar1, M[i][j], S[i][j][1]);
            }
          }
      }
      // column stage of At.m.A
      const T ac0 = (T)c_at[pc][0][b], ac1 = (T)c_at[pc][1][b];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j)
#pragma unroll
          for (int ii = 0; ii < 2; ++ii) {
            if (b == 0) {
              Tt[i][j][ii][0] = mul_rn(S[i][j][ii], ac0);
              Tt[i][j][ii][1] = mul_rn(S[i][j][ii], ac1);
            } else {
              Tt[i][j][ii][0] = fma_rn(S[i][j][ii], ac0, Tt[i][j][ii][0]);
              Tt[i][j][ii][1] = fma_rn(S[i][j][ii], ac1, Tt[i][j][ii][1]);
            }
          }
    }
    // aggregation in plan order
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j)
#pragma unroll
        for (int ii = 0; ii < 2; ++ii)
#pragma unroll
          for (int jj = 0; jj < 2; ++jj)
            acc[i][j][ii][jj] = (p == 0) ? Tt[i][j][ii][jj] : add_rn(acc[i][j][ii][jj], Tt[i][j][ii][jj]);
    fq_base += lr * lc;
  }

  // epilogue: interleave 2x2 tiles into NCHW and truncate odd extents
  bool bad = false;
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int64_t tile = tile0 + tm * TM + i;
    if (tile >= tiles) continue;
    const int tx = (int)(tile % d.tw);
    const int64_t t2 = tile / d.tw;
    const int ty = (int)(t2 % d.th);
    const int n = (int)(t2 / d.th);
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int f = f0 + tn * TN + j;
      if (f >= F) continue;
      T* yf = y + ((int64_t)n * F + f) * d.oh * d.ow;
#pragma unroll
      for (int ii = 0; ii < 2; ++ii)
#pragma unroll
        for (int jj = 0; jj < 2; ++jj) {
          const int oy = 2 * ty + ii, ox = 2 * tx + jj;
          if (oy < d.oh && ox < d.ow) {
            const T v = acc[i][j][ii][jj];
            bad |= !isfinite(v);
            yf[(int64_t)oy * d.ow + ox] = v;
          }
        }
    }
  }
  if (bad && flag) *flag = 1;
}

// binary32 variant with packed f32x2 arithmetic (FFMA2/FMUL2/FADD2): the
// same per-lane operations in the same order as gemm_exact_kernel<float>
// (so the same bits), two filters per instruction.
template <int BM, int BN, int TM, int TN, int KC>
__global__ void __launch_bounds__((BM / TM) * (BN / TN))
gemm_exact_f32x2_kernel(const dwm_desc_t d, const float* __restrict__ V, const float* __restrict__ U,
                        float* __restrict__ y, int32_t* __restrict__ flag) {
  constexpr int GM = BM / TM, GN = BN / TN, NT = GM * GN, NP = TN / 2, VW = 4;
  static_assert(TM == 4 && TN == 4, "one 16-byte smem load per operand and k");
  __shared__ __align__(16) float sV[KC][BM];
  __shared__ __align__(16) float sU[KC][BN];
  const int tid = threadIdx.x;
  const int tm = tid % GM, tn = tid / GM;
  const int64_t tile0 = (int64_t)blockIdx.x * BM;
  const int f0 = blockIdx.y * BN;
  const int C = d.c, F = d.f;
  const int64_t tiles = d.tiles;
  const bool vec = (C % VW) == 0;

  f2 acc[TM][NP][2][2], Tt[TM][NP][2][2], S[TM][NP][2];
  int fq_base = 0;
  for (int p = 0; p < d.n_row_parts * d.n_col_parts; ++p) {
    const int pr = d.row_parts[p / d.n_col_parts].count;
    const int pc = d.col_parts[p % d.n_col_parts].count;
    const int lr = pr + 1, lc = pc + 1;
    for (int b = 0; b < lc; ++b) {
      for (int a = 0; a < lr; ++a) {
        const int fq = fq_base + a * lc + b;
        const float* Vq = V + (int64_t)fq * tiles * C;
        const float* Uq = U + (int64_t)fq * F * C;
        f2 M[TM][NP];
        for (int k0 = 0; k0 < C; k0 += KC) {
          const int kn = min(KC, C - k0);
          __syncthreads();
          if (vec) {
            for (int e = tid; e < BM * (KC / VW); e += NT) {
              const int kq = e % (KC / VW), t = e / (KC / VW);
              const int64_t tile = tile0 + t;
              float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
              if (tile < tiles && k0 + kq * VW < C) q = __ldg(reinterpret_cast<const float4*>(Vq + tile * C + k0 + kq * VW));
              sV[kq * VW + 0][t] = q.x; sV[kq * VW + 1][t] = q.y; sV[kq * VW + 2][t] = q.z; sV[kq * VW + 3][t] = q.w;
            }
            for (int e = tid; e < BN * (KC / VW); e += NT) {
              const int kq = e % (KC / VW), fl = e / (KC / VW);
              float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
              if (f0 + fl < F && k0 + kq * VW < C)
                q = __ldg(reinterpret_cast<const float4*>(Uq + (int64_t)(f0 + fl) * C + k0 + kq * VW));
              sU[kq * VW + 0][fl] = q.x; sU[kq * VW + 1][fl] = q.y; sU[kq * VW + 2][fl] = q.z; sU[kq * VW + 3][fl] = q.w;
            }
          } else {
            for (int e = tid; e < BM * KC; e += NT) {
              const int k = e % KC, t = e / KC;
              const int64_t tile = tile0 + t;
              sV[k][t] = (k < kn && tile < tiles) ? Vq[tile * C + k0 + k] : 0.f;
            }
            for (int e = tid; e < BN * KC; e += NT) {
              const int k = e % KC, fl = e / KC;
              sU[k][fl] = (k < kn && f0 + fl < F) ? Uq[(int64_t)(f0 + fl) * C + k0 + k] : 0.f;
            }
          }
          __syncthreads();
          for (int k = 0; k < kn; ++k) {
            const float4 vq = *reinterpret_cast<const float4*>(&sV[k][tm * TM]);
            const float4 uq = *reinterpret_cast<const float4*>(&sU[k][tn * TN]);
            const float vv[TM] = {vq.x, vq.y, vq.z, vq.w};
            const f2 u2[NP] = {pk(uq.x, uq.y), pk(uq.z, uq.w)};
            if (k0 + k == 0) {
#pragma unroll
              for (int i = 0; i < TM; ++i)
#pragma unroll
                for (int jp = 0; jp < NP; ++jp) M[i][jp] = mul2(u2[jp], pk(vv[i], vv[i]));
            } else {
#pragma unroll
              for (int i = 0; i < TM; ++i)
#pragma unroll
                for (int jp = 0; jp < NP; ++jp) M[i][jp] = fma2(u2[jp], pk(vv[i], vv[i]), M[i][jp]);
            }
          }
        }
        const f2 ar0 = pk(c_at[pr][0][a], c_at[pr][0][a]), ar1 = pk(c_at[pr][1][a], c_at[pr][1][a]);
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int jp = 0; jp < NP; ++jp) {
            if (a == 0) {
              S[i][jp][0] = mul2(ar0, M[i][jp]);
              S[i][jp][1] = mul2(ar1, M[i][jp]);
            } else {
              S[i][jp][0] = fma2(ar0, M[i][jp], S[i][jp][0]);
              S[i][jp][1] = fma2(ar1, M[i][jp], S[i][jp][1]);
            }
          }
      }
      const f2 ac0 = pk(c_at[pc][0][b], c_at[pc][0][b]), ac1 = pk(c_at[pc][1][b], c_at[pc][1][b]);
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int jp = 0; jp < NP; ++jp)
#pragma unroll
          for (int ii = 0; ii < 2; ++ii) {
            if (b == 0) {
              Tt[i][jp][ii][0] = mul2(S[i][jp][ii], ac0);
              Tt[i][jp][ii][1] = mul2(S[i][jp][ii], ac1);
            } else {
              Tt[i][jp][ii][0] = fma2(S[i][jp][ii], ac0, Tt[i][jp][ii][0]);
              Tt[i][jp][ii][1] = fma2(S[i][jp][ii], ac1, Tt[i][jp][ii][1]);
            }
          }
    }
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int jp = 0; jp < NP; ++jp)
#pragma unroll
        for (int ii = 0; ii < 2; ++ii)
#pragma unroll
          for (int jj = 0; jj < 2; ++jj)
            acc[i][jp][ii][jj] = (p == 0) ? Tt[i][jp][ii][jj] : add2(acc[i][jp][ii][jj], Tt[i][jp][ii][jj]);
    fq_base += lr * lc;
  }

  bool bad = false;
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int64_t tile = tile0 + tm * TM + i;
    if (tile >= tiles) continue;
    const int tx = (int)(tile % d.tw);
    const int64_t t2 = tile / d.tw;
    const int ty = (int)(t2 % d.th);
    const int n = (int)(t2 / d.th);
#pragma unroll
    for (int jp = 0; jp < NP; ++jp)
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        const int f = f0 + tn * TN + 2 * jp + half;
        if (f >= F) continue;
        float* yf = y + ((int64_t)n * F + f) * d.oh * d.ow;
#pragma unroll
        for (int ii = 0; ii < 2; ++ii)
#pragma unroll
          for (int jj = 0; jj < 2; ++jj) {
            const int oy = 2 * ty + ii, ox = 2 * tx + jj;
            if (oy < d.oh && ox < d.ow) {
              const float2 v2 = upk(acc[i][jp][ii][jj]);
              const float v = half ? v2.y : v2.x;
              bad |= !isfinite(v);
              yf[(int64_t)oy * d.ow + ox] = v;
            }
          }
      }
  }
  if (bad && flag) *flag = 1;
}

int launch_gemm_exact(const dwm_desc_t& d, int dtype, const void* V, const void* U, void* y,
                      int32_t* flag, cudaStream_t s) {
  if (dtype == DWM_F64) {
    constexpr int BM = 32, BN = 64, TM = 2, TN = 4, KC = 16;
    const dim3 grid((unsigned)((d.tiles + BM - 1) / BM), (unsigned)((d.f + BN - 1) / BN));
    gemm_exact_kernel<double, BM, BN, TM, TN, KC><<<grid, (BM / TM) * (BN / TN), 0, s>>>(
        d, (const double*)V, (const double*)U, (double*)y, flag);
  } else {
    constexpr int BM = 64, BN = 64, TM = 4, TN = 4, KC = 16;
    const int64_t ctas = ((d.tiles + BM - 1) / BM) * ((d.f + BN - 1) / BN);
    if (ctas < 148) {
      // small problem (e.g. one 56x56 image): one output per thread, 16x16
      // blocks, so the work spreads over the SMs instead of a handful of CTAs
      constexpr int SB = 16;
#ifndef DWM_EXACT_SMALL_KC
#define DWM_EXACT_SMALL_KC 32
#endif
      // deeper K chunks: each chunk is a load -> barrier -> FMA round trip,
      // which is what bounds a problem this small (same summation order)
      constexpr int SKC = DWM_EXACT_SMALL_KC;
      const dim3 g2((unsigned)((d.tiles + SB - 1) / SB), (unsigned)((d.f + SB - 1) / SB));
      gemm_exact_kernel<float, SB, SB, 1, 1, SKC><<<g2, SB * SB, 0, s>>>(
          d, (const float*)V, (const float*)U, (float*)y, flag);
    } else {
      const dim3 grid((unsigned)((d.tiles + BM - 1) / BM), (unsigned)((d.f + BN - 1) / BN));
      gemm_exact_f32x2_kernel<BM, BN, TM, TN, KC><<<grid, (BM / TM) * (BN / TN), 0, s>>>(
          d, (const float*)V, (const float*)U, (float*)y, flag);
    }
  }
  DWM_CUDA_TRY(cudaGetLastError());
  return DWM_OK;
}

}  // namespace dwm
