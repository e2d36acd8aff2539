#pragma once
// dwm_small_c.cuh -- fully fused DWM forward for small input-channel counts
// (C_in <= 4: the ResNet-50 / AlexNet stems of BASELINE configs[1], [2]).
//
// With K = C_in <= 4 the per-frequency "GEMM" is not a tensor-core
// contraction (SURVEY §7 hard part 4); the whole forward is FP32-pipe bound
// (FP32 FMA peak on B200 = 148 SM x 128 lanes x 1.965 GHz, measured 72 TFLOP/s
// with tools/fp32_peak.cu).  One persistent kernel does everything on the CUDA
// cores and only x is read and y written in HBM:
//
//   prologue : U[freq][F][C] (from the filter-transform kernel) -> smem,
//              transposed to [freq][C][f-block] (resident for the whole kernel).
//   per tile block (BM consecutive 2x2 output tiles) and per plan part:
//     producer: polyphase gather of the part's (count+1)^2 input window for
//               every (tile, channel) straight from x (padding and the
//               reference's even-extension zeros by predicate), Bt.d.B row
//               stage then column stage with compile-time coefficients ->
//               V part in smem [q][c][tile] (double buffered; the x loads of
//               part p+1 are issued before part p's math).
//     consumer: per frequency, M = sum_c U*V (FMA chain, c ascending);
//               At.m.A row stage S, column stage T with compile-time
//               coefficients (0 skipped, +-1 as add/sub); y += T in plan
//               order, y accumulated in shared memory.  All of it runs on
//               packed f32x2 FFMA2/FADD2 pairs over adjacent filters, which
//               halves FP32 issue slots (each lane of a pair is an ordinary
//               IEEE binary32 RN operation).
//   epilogue : interleave the 2x2 tiles into NCHW, truncate odd extents,
//              raise the non-finite flag.
//
// Every rounding step is the reference's (engines.py:164-194, 244-255 with a
// sequential BLAS), so the output equals the reference DWM in binary32 (see
// tests/test_gpu_parity.py; only the sign of exact zeros may differ).
#include <utility>

#include "dwm_common.cuh"
#include <cstdlib>
#include <cstring>
#include "dwm_kernels.h"
#include "dwm_wino.cuh"

namespace dwm {
namespace smallc {

using namespace wino;

constexpr int THREADS = 256;  // 32 tile lanes x 8 filter groups
constexpr int MAXQ = 16;      // frequencies per part, (3+1)^2

// every At row starts with +1, so no sign tracking is needed here
template <int K, bool FIRST> __device__ __forceinline__ void chain2(f2& acc, f2 m) {
  if constexpr (K == 0) return;
  else if constexpr (FIRST) { static_assert(K == 1, "At rows start with +1"); acc = m; }
  else if constexpr (K == 1) acc = add2(acc, m);
  else acc = sub2(acc, m);
}

template <int CC_, int TM_, int TN_, int MINB_ = 1>
struct Cfg {
  static constexpr int CC = CC_, TM = TM_, TN = TN_, MINB = MINB_;
  static constexpr int BM = 32 * TM;         // tiles per block
  static constexpr int BN = 8 * TN;          // filters per block
  static constexpr int NP = TN / 2;          // filter pairs per thread
  static constexpr int NACC2 = TM * NP * 4;  // packed accumulators per thread
  static constexpr int VSTAGE = MAXQ * CC * BM;
  static size_t smem_bytes(int num_freqs) {
    return ((size_t)NACC2 * 2 * THREADS + 2 * (size_t)VSTAGE + (size_t)num_freqs * CC * BN) * sizeof(float);
  }
};

// Consume one part.  sV: [q][CC][BM]; sU: part's first frequency, [q][CC][BN];
// sAcc: packed y accumulators [NACC2][THREADS] (conflict-free 8-byte slots).
template <class K, int PR, int PC>
__device__ __forceinline__ void consume_part(const float* __restrict__ sV, const float* __restrict__ sU,
                                             f2* __restrict__ sAcc, int tid, bool first_part) {
  constexpr int LR = PR + 1, LC = PC + 1, TM = K::TM, NP = K::NP, CC = K::CC, BM = K::BM, BN = K::BN;
  const int tm = tid % 32, tn = tid / 32;
  f2 T[TM][NP][2][2];
  static_for<LC>([&](auto bI) {
    constexpr int b = decltype(bI)::value;
    f2 S[TM][NP][2];
    static_for<LR>([&](auto aI) {
      constexpr int a = decltype(aI)::value;
      constexpr int q = a * LC + b;
      f2 M[TM][NP];
#pragma unroll
      for (int c = 0; c < CC; ++c) {
        float v[TM];
#pragma unroll
        for (int i = 0; i < TM; ++i) v[i] = sV[(q * CC + c) * BM + tm + 32 * i];
        f2 u[NP];
        const float* up = sU + (q * CC + c) * BN + tn * K::TN;
#pragma unroll
        for (int jp = 0; jp < NP; jp += 2) {
          // 16-byte loads need the thread's filter offset tn*TN 16-byte aligned
          if (K::TN % 4 == 0 && jp + 1 < NP) {
            const float4 u4 = *reinterpret_cast<const float4*>(up + 2 * jp);
            u[jp] = pk(u4.x, u4.y);
            u[jp + 1] = pk(u4.z, u4.w);
          } else {
            const float2 u2 = *reinterpret_cast<const float2*>(up + 2 * jp);
            u[jp] = pk(u2.x, u2.y);
            if (jp + 1 < NP) {
              const float2 u3 = *reinterpret_cast<const float2*>(up + 2 * jp + 2);
              u[jp + 1] = pk(u3.x, u3.y);
            }
          }
        }
#pragma unroll
        for (int i = 0; i < TM; ++i) {
          const f2 vv = pk(v[i], v[i]);
#pragma unroll
          for (int jp = 0; jp < NP; ++jp) M[i][jp] = (c == 0) ? mul2(u[jp], vv) : fma2(u[jp], vv, M[i][jp]);
        }
      }
      // row stage of At.m.A: S[i'] = sum_a At_r[i'][a] M_a
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int jp = 0; jp < NP; ++jp) {
          chain2<at_coef(PR, 0, a), (a == at_first(PR, 0))>(S[i][jp][0], M[i][jp]);
          chain2<at_coef(PR, 1, a), (a == at_first(PR, 1))>(S[i][jp][1], M[i][jp]);
        }
    });
    // column stage: T[i'][j'] = sum_b S[i'](b) * At_c[j'][b]
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int jp = 0; jp < NP; ++jp)
#pragma unroll
        for (int ii = 0; ii < 2; ++ii) {
          chain2<at_coef(PC, 0, b), (b == at_first(PC, 0))>(T[i][jp][ii][0], S[i][jp][ii]);
          chain2<at_coef(PC, 1, b), (b == at_first(PC, 1))>(T[i][jp][ii][1], S[i][jp][ii]);
        }
  });
  // aggregation in plan order (tensor.py:68-81): acc = acc + T
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int jp = 0; jp < NP; ++jp)
#pragma unroll
      for (int ii = 0; ii < 2; ++ii)
#pragma unroll
        for (int jj = 0; jj < 2; ++jj) {
          f2* slot = sAcc + (((i * NP + jp) * 2 + ii) * 2 + jj) * THREADS + tid;
          *slot = first_part ? T[i][jp][ii][jj] : add2(*slot, T[i][jp][ii][jj]);
        }
}

// Producer geometry of one (tile, channel) for a tile block, computed once.
struct ProdTile {
  const float* xc;  // x[n][c]
  int y0, x0;       // 2*ty*s_h - pad_top, 2*tx*s_w - pad_left
  int ky, kx;       // 2*ty, 2*tx (window sample index base)
  bool live;
};

__device__ __forceinline__ ProdTile prod_tile(const dwm_desc_t& d, const float* __restrict__ x, int tile, int c) {
  ProdTile p;
  p.live = tile < d.tiles;
  const int t = p.live ? tile : 0;
  const int tx = t % d.tw;
  const int t2 = t / d.tw;
  const int ty = t2 % d.th;
  const int n = t2 / d.th;
  p.xc = x + ((size_t)n * d.c + c) * (size_t)d.h * d.w;
  p.ky = 2 * ty;
  p.kx = 2 * tx;
  p.y0 = 2 * ty * d.s_h - d.pad_top;
  p.x0 = 2 * tx * d.s_w - d.pad_left;
  return p;
}

// Producer half 1: gather the part's (count+1)^2 window into registers.
__device__ __forceinline__ void load_window(const dwm_desc_t& d, const ProdTile& p, int rp, int cp,
                                            float win[4][4]) {
  const dwm_axis_part_t R = d.row_parts[rp], Cc = d.col_parts[cp];
  int rows[4], cols[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int row = p.y0 + R.origin + d.s_h * i;
    rows[i] = (p.live && i <= R.count && p.ky + i < d.oh - 1 + R.count && row >= 0 && row < d.h) ? row * d.w : -1;
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int col = p.x0 + Cc.origin + d.s_w * j;
    cols[j] = (j <= Cc.count && p.kx + j < d.ow - 1 + Cc.count && col >= 0 && col < d.w) ? col : -1;
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
      win[i][j] = (rows[i] >= 0 && cols[j] >= 0) ? __ldg(p.xc + rows[i] + cols[j]) : 0.f;
}

// Producer half 2: Bt.d.B with compile-time coefficients -> sV[q][c][t].
template <class K, int PR, int PC>
__device__ __forceinline__ void transform_store(const float (&win)[4][4], float* __restrict__ sV, int t, int c) {
  input_transform_part<PR, PC>(win, [&](int q, float v) { sV[(q * K::CC + c) * K::BM + t] = v; });
}

template <class K>
__global__ void __launch_bounds__(THREADS, K::MINB)
small_c_kernel(const dwm_desc_t d, const float* __restrict__ x, const float* __restrict__ U,
               float* __restrict__ y, int32_t* __restrict__ flag) {
  constexpr int CC = K::CC, BM = K::BM, BN = K::BN, TM = K::TM, TN = K::TN, NP = K::NP;
  extern __shared__ __align__(16) float smem[];
  f2* sAcc = reinterpret_cast<f2*>(smem);                      // [NACC2][THREADS]
  float* sVbuf = smem + K::NACC2 * 2 * THREADS;                  // [2][MAXQ][CC][BM]
  float* sU = sVbuf + 2 * K::VSTAGE;                             // [freq][CC][BN]

  const int tid = threadIdx.x;
  const int tm = tid % 32, tn = tid / 32;
  const int f0 = blockIdx.y * BN;
  const int F = d.f;
  const int nparts = d.n_row_parts * d.n_col_parts;
  const int nblocks = (int)((d.tiles + BM - 1) / BM);

  for (int e = tid; e < d.num_freqs * CC * BN; e += THREADS) {
    const int fl = e % BN, c = (e / BN) % CC, q = e / (BN * CC);
    const int f = f0 + fl;
    sU[e] = f < F ? U[((size_t)q * F + f) * CC + c] : 0.f;
  }

  // producer slots: (tile t, channel c), t fastest within a warp
  constexpr int PSLOTS = BM * CC;
  constexpr int PPER = (PSLOTS + THREADS - 1) / THREADS;  // slots per thread (1 or 2)
  int pt[PPER], pch[PPER];
  bool pact[PPER];
#pragma unroll
  for (int s = 0; s < PPER; ++s) {
    const int e = tid + s * THREADS;
    pact[s] = e < PSLOTS;
    pt[s] = e % BM;
    pch[s] = pact[s] ? e / BM : 0;
  }

  int tb = blockIdx.x;
  if (tb >= nblocks) return;
  float win[PPER][4][4];
  ProdTile ptile[PPER];
#pragma unroll
  for (int s = 0; s < PPER; ++s) {
    ptile[s] = prod_tile(d, x, tb * BM + pt[s], pch[s]);
    if (pact[s]) {
      load_window(d, ptile[s], 0, 0, win[s]);
#define DWM_TS0(A, B) transform_store<K, A, B>(win[s], sVbuf, pt[s], pch[s])
      DWM_PART_SWITCH(d.row_parts[0].count, d.col_parts[0].count, DWM_TS0)
#undef DWM_TS0
    }
  }
  __syncthreads();

  int stage = 0;
  for (; tb < nblocks; tb += gridDim.x) {
    int qoff = 0;
    for (int p = 0; p < nparts; ++p) {
      const int rp = p / d.n_col_parts, cpi = p % d.n_col_parts;
      // next unit of work: part p+1 of this block, or part 0 of the next block
      const bool last = p + 1 == nparts;
      const bool has_next = !last || (tb + (int)gridDim.x < nblocks);
      const int np = last ? 0 : p + 1;
      const int nrp = np / d.n_col_parts, ncp = np % d.n_col_parts;
#pragma unroll
      for (int s = 0; s < PPER; ++s) {
        if (last && has_next) ptile[s] = prod_tile(d, x, (tb + gridDim.x) * BM + pt[s], pch[s]);
        if (pact[s] && has_next) load_window(d, ptile[s], nrp, ncp, win[s]);
      }

      const float* sV = sVbuf + stage * K::VSTAGE;
      const float* sUp = sU + qoff * CC * BN;
#define DWM_CONSUME(A, B) consume_part<K, A, B>(sV, sUp, sAcc, tid, p == 0)
      DWM_PART_SWITCH(d.row_parts[rp].count, d.col_parts[cpi].count, DWM_CONSUME)
#undef DWM_CONSUME
      qoff += (d.row_parts[rp].count + 1) * (d.col_parts[cpi].count + 1);

      if (has_next) {
        float* sVn = sVbuf + (stage ^ 1) * K::VSTAGE;
#pragma unroll
        for (int s = 0; s < PPER; ++s) {
          if (!pact[s]) continue;
#define DWM_TSN(A, B) transform_store<K, A, B>(win[s], sVn, pt[s], pch[s])
          DWM_PART_SWITCH(d.row_parts[nrp].count, d.col_parts[ncp].count, DWM_TSN)
#undef DWM_TSN
        }
      }
      stage ^= 1;
      __syncthreads();
    }
    // epilogue: 2x2 tiles -> NCHW
    bool bad = false;
#pragma unroll
    for (int i = 0; i < TM; ++i) {
      const int tile = tb * BM + tm + 32 * i;
      if (tile >= d.tiles) continue;
      const int tx = tile % d.tw;
      const int t2 = tile / d.tw;
      const int ty = t2 % d.th;
      const int n = t2 / d.th;
#pragma unroll
      for (int jp = 0; jp < NP; ++jp) {
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          const int f = f0 + tn * TN + 2 * jp + half;
          if (f >= F) continue;
          float* yf = y + ((size_t)n * F + f) * (size_t)d.oh * d.ow;
#pragma unroll
          for (int ii = 0; ii < 2; ++ii) {
            const int oy = 2 * ty + ii;
            if (oy >= d.oh) continue;
            const float2 a0 = upk(sAcc[(((i * NP + jp) * 2 + ii) * 2 + 0) * THREADS + tid]);
            const float2 a1 = upk(sAcc[(((i * NP + jp) * 2 + ii) * 2 + 1) * THREADS + tid]);
            const float v0 = half ? a0.y : a0.x, v1 = half ? a1.y : a1.x;
            const int ox = 2 * tx;
            float* dst = yf + (size_t)oy * d.ow + ox;
            if (ox + 1 < d.ow) {
              bad |= !(isfinite(v0) && isfinite(v1));
              if ((d.ow & 1) == 0 && ((uintptr_t)y & 7) == 0) {
                __stcs(reinterpret_cast<float2*>(dst), make_float2(v0, v1));
              } else {
                __stcs(dst, v0);
                __stcs(dst + 1, v1);
              }
            } else {
              bad |= !isfinite(v0);
              __stcs(dst, v0);
            }
          }
        }
      }
    }
    if (bad && flag) *flag = 1;
  }
}

// ===========================================================================
// Warp-specialized variant (round 2): 4 producer warps gather + transform V
// into a 3-stage shared-memory ring; 8 consumer warps run the channel FMA
// chains and the At stages with the y accumulators in REGISTERS (no shared-
// memory read-modify-write per part, no __syncthreads: mbarrier handshakes),
// register budgets redistributed with setmaxnreg.  Same arithmetic in the
// same order as small_c_kernel, so the same bits (the reference's).
// ===========================================================================
#ifndef DWM_WS_PROD
#define DWM_WS_PROD 8  // producer warps (8: cfg2 -3 %, cfg3 -7 % vs 4, profiles/r2/ab_small_c_producers.txt)
#endif
constexpr int WS_CONS = 8, WS_PROD = DWM_WS_PROD, WS_THREADS = 32 * (WS_CONS + WS_PROD);
constexpr int WS_STAGES = 3;
constexpr int WS_REG_CONS = 208, WS_REG_PROD = WS_PROD == 4 ? 80 : 48;  // 8 x 32 x (208 + 48) = 65536
static_assert(WS_CONS * 32 * WS_REG_CONS + WS_PROD * 32 * WS_REG_PROD <= 65536, "register file");

template <int CC_, int TM_, int TN_>
struct WsCfg {
  static constexpr int CC = CC_, TM = TM_, TN = TN_;
  static constexpr int BM = 32 * TM;   // tiles per block (lane = tile)
  static constexpr int BN = 8 * TN;    // filters per block (consumer warp = filter group)
  static constexpr int NP = TN / 2;
  static constexpr int VSTAGE = MAXQ * CC * BM;
  static constexpr int PPER = (BM * CC + 32 * WS_PROD - 1) / (32 * WS_PROD);  // producer slots per thread
  static size_t smem_bytes(int num_freqs) {
    return (WS_STAGES * (size_t)VSTAGE + (size_t)num_freqs * CC * BN) * sizeof(float) + 2 * WS_STAGES * 8 + 16;
  }
};

// consume_part with the plan-order aggregation into register accumulators
template <class K, int PR, int PC>
__device__ __forceinline__ void consume_part_reg(const float* __restrict__ sV, const float* __restrict__ sU,
                                                 f2 (&acc)[K::TM][K::NP][2][2], int tm, int tn, bool first_part) {
  constexpr int LR = PR + 1, LC = PC + 1, TM = K::TM, NP = K::NP, CC = K::CC, BM = K::BM, BN = K::BN;
  f2 T[TM][NP][2][2];
  static_for<LC>([&](auto bI) {
    constexpr int b = decltype(bI)::value;
    f2 S[TM][NP][2];
    static_for<LR>([&](auto aI) {
      constexpr int a = decltype(aI)::value;
      constexpr int q = a * LC + b;
      f2 M[TM][NP];
#pragma unroll
      for (int c = 0; c < CC; ++c) {
        float v[TM];
#pragma unroll
        for (int i = 0; i < TM; ++i) v[i] = sV[(q * CC + c) * BM + tm + 32 * i];
        f2 u[NP];
        const float* up = sU + (q * CC + c) * BN + tn * K::TN;
#pragma unroll
        for (int jp = 0; jp < NP; jp += 2) {
          if (K::TN % 4 == 0 && jp + 1 < NP) {
            const float4 u4 = *reinterpret_cast<const float4*>(up + 2 * jp);
            u[jp] = pk(u4.x, u4.y);
            u[jp + 1] = pk(u4.z, u4.w);
          } else {
            const float2 u2 = *reinterpret_cast<const float2*>(up + 2 * jp);
            u[jp] = pk(u2.x, u2.y);
            if (jp + 1 < NP) {
              const float2 u3 = *reinterpret_cast<const float2*>(up + 2 * jp + 2);
              u[jp + 1] = pk(u3.x, u3.y);
            }
          }
        }
#pragma unroll
        for (int i = 0; i < TM; ++i) {
          const f2 vv = pk(v[i], v[i]);
#pragma unroll
          for (int jp = 0; jp < NP; ++jp) M[i][jp] = (c == 0) ? mul2(u[jp], vv) : fma2(u[jp], vv, M[i][jp]);
        }
      }
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int jp = 0; jp < NP; ++jp) {
          chain2<at_coef(PR, 0, a), (a == at_first(PR, 0))>(S[i][jp][0], M[i][jp]);
          chain2<at_coef(PR, 1, a), (a == at_first(PR, 1))>(S[i][jp][1], M[i][jp]);
        }
    });
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int jp = 0; jp < NP; ++jp)
#pragma unroll
        for (int ii = 0; ii < 2; ++ii) {
          chain2<at_coef(PC, 0, b), (b == at_first(PC, 0))>(T[i][jp][ii][0], S[i][jp][ii]);
          chain2<at_coef(PC, 1, b), (b == at_first(PC, 1))>(T[i][jp][ii][1], S[i][jp][ii]);
        }
  });
  // aggregation in plan order (tensor.py:68-81): acc = acc + T
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int jp = 0; jp < NP; ++jp)
#pragma unroll
      for (int ii = 0; ii < 2; ++ii)
#pragma unroll
        for (int jj = 0; jj < 2; ++jj)
          acc[i][jp][ii][jj] = first_part ? T[i][jp][ii][jj] : add2(acc[i][jp][ii][jj], T[i][jp][ii][jj]);
}

template <uint32_t N>
__device__ __forceinline__ void ws_setmaxnreg_inc() { asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(N)); }
template <uint32_t N>
__device__ __forceinline__ void ws_setmaxnreg_dec() { asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(N)); }

__device__ __forceinline__ void ws_bar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void ws_bar_arrive(uint64_t* bar) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(bar))
               : "memory");
}
__device__ __forceinline__ void ws_bar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(bar);
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok)
                 : "r"(a), "r"(parity)
                 : "memory");
}

// Plan signatures the warp-specialized kernel is compiled for part by part
// (square plans: the same tap-count sequence on both axes).  With the part
// sequence known at compile time, each part's FMA chains, At stages and the
// plan-order aggregation inline into one straight line: no runtime part
// switch, and the y accumulators stay in the same registers across parts
// (the generic loop moves them at every switch).  SIG 0 = generic.
template <int SIG> struct PlanSig { static constexpr int n = 0; static constexpr int c[4] = {0, 0, 0, 0}; };
template <> struct PlanSig<1> { static constexpr int n = 3; static constexpr int c[4] = {3, 1, 3, 0}; };  // 7x7/2
// (the 16-part 11x11/4 sequence was measured slower unrolled: cfg3 1.32 -> 1.55 ms)
template <int SIG>
__host__ __device__ constexpr int sig_qoff(int p) {  // first frequency of part p (row-major parts)
  int q = 0;
  for (int i = 0; i < p; ++i) q += (PlanSig<SIG>::c[i / PlanSig<SIG>::n] + 1) * (PlanSig<SIG>::c[i % PlanSig<SIG>::n] + 1);
  return q;
}
inline int match_plan_sig(const dwm_desc_t& d) {
  auto axis_is = [&](const dwm_axis_part_t* parts, int n, auto sig) {
    using S = decltype(sig);
    if (n != S::n) return false;
    for (int i = 0; i < n; ++i)
      if (parts[i].count != S::c[i]) return false;
    return true;
  };
  if (axis_is(d.row_parts, d.n_row_parts, PlanSig<1>{}) && axis_is(d.col_parts, d.n_col_parts, PlanSig<1>{})) return 1;
  return 0;
}

template <class K, int SIG>
__global__ void __launch_bounds__(WS_THREADS, 1)
small_c_ws_kernel(const dwm_desc_t d, const float* __restrict__ x, const float* __restrict__ U,
                  float* __restrict__ y, int32_t* __restrict__ flag) {
  constexpr int CC = K::CC, BM = K::BM, BN = K::BN, TM = K::TM, TN = K::TN, NP = K::NP;
  extern __shared__ __align__(16) float smem[];
  float* sVbuf = smem;                                   // [STAGES][MAXQ][CC][BM]
  float* sU = sVbuf + WS_STAGES * K::VSTAGE;             // [freq][CC][BN]
  uint64_t* full = reinterpret_cast<uint64_t*>(
      (reinterpret_cast<uintptr_t>(sU + (size_t)d.num_freqs * CC * BN) + 7) & ~(uintptr_t)7);
  uint64_t* empty = full + WS_STAGES;

  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const int f0 = blockIdx.y * BN;
  const int F = d.f;
  const int nparts = d.n_row_parts * d.n_col_parts;
  const int nblocks = (int)((d.tiles + BM - 1) / BM);

  for (int e = tid; e < d.num_freqs * CC * BN; e += WS_THREADS) {
    const int fl = e % BN, c = (e / BN) % CC, q = e / (BN * CC);
    const int f = f0 + fl;
    sU[e] = f < F ? U[((size_t)q * F + f) * CC + c] : 0.f;
  }
  if (tid == 0) {
    for (int i = 0; i < WS_STAGES; ++i) {
      ws_bar_init(&full[i], WS_PROD);
      ws_bar_init(&empty[i], WS_CONS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp >= WS_CONS) {
    ws_setmaxnreg_dec<WS_REG_PROD>();
    // ================= producers: window gather + Bt.d.B -> V stage =================
    const int ptid = tid - 32 * WS_CONS;
    int pt[K::PPER], pch[K::PPER];
    bool pact[K::PPER];
#pragma unroll
    for (int s = 0; s < K::PPER; ++s) {
      const int e = ptid + s * 32 * WS_PROD;
      pact[s] = e < BM * CC;
      pt[s] = e % BM;
      pch[s] = pact[s] ? e / BM : 0;
    }
    uint32_t it = 0;
    for (int tb = blockIdx.x; tb < nblocks; tb += gridDim.x) {
      ProdTile ptile[K::PPER];
#pragma unroll
      for (int s = 0; s < K::PPER; ++s) ptile[s] = prod_tile(d, x, tb * BM + pt[s], pch[s]);
      auto produce = [&](int rp, int cp, auto store) {
        const uint32_t st = it % WS_STAGES;
        float win[K::PPER][4][4];
#pragma unroll
        for (int s = 0; s < K::PPER; ++s)
          if (pact[s]) load_window(d, ptile[s], rp, cp, win[s]);
        ws_bar_wait(&empty[st], ((it / WS_STAGES) & 1) ^ 1);
        float* sV = sVbuf + st * K::VSTAGE;
#pragma unroll
        for (int s = 0; s < K::PPER; ++s)
          if (pact[s]) store(win[s], sV, pt[s], pch[s]);
        __syncwarp();
        if (lane == 0) ws_bar_arrive(&full[st]);
        ++it;
      };
      // (the producer stays generic: its unrolled part sequence spilled at 48 registers)
      for (int p = 0; p < nparts; ++p) {
        const int rp = p / d.n_col_parts, cp = p % d.n_col_parts;
        produce(rp, cp, [&](const float (&w)[4][4], float* sV, int t, int c) {
#define DWM_WSTS(A, B) transform_store<K, A, B>(w, sV, t, c)
          DWM_PART_SWITCH(d.row_parts[rp].count, d.col_parts[cp].count, DWM_WSTS)
#undef DWM_WSTS
        });
      }
    }
  } else {
    ws_setmaxnreg_inc<WS_REG_CONS>();
    // ================= consumers: FMA chains, At stages, register accumulators =================
    const int tm = lane, tn = warp;
    f2 acc[TM][NP][2][2];
    uint32_t it = 0;
    for (int tb = blockIdx.x; tb < nblocks; tb += gridDim.x) {
      if constexpr (SIG == 0) {
        int qoff = 0;
        for (int p = 0; p < nparts; ++p, ++it) {
          const int rp = p / d.n_col_parts, cpi = p % d.n_col_parts;
          const uint32_t st = it % WS_STAGES;
          ws_bar_wait(&full[st], (it / WS_STAGES) & 1);
          const float* sV = sVbuf + st * K::VSTAGE;
          const float* sUp = sU + qoff * CC * BN;
#define DWM_WSC(A, B) consume_part_reg<K, A, B>(sV, sUp, acc, tm, tn, p == 0)
          DWM_PART_SWITCH(d.row_parts[rp].count, d.col_parts[cpi].count, DWM_WSC)
#undef DWM_WSC
          __syncwarp();
          if (lane == 0) ws_bar_arrive(&empty[st]);
          qoff += (d.row_parts[rp].count + 1) * (d.col_parts[cpi].count + 1);
        }
      } else {
        using S = PlanSig<SIG>;
        static_for<S::n * S::n>([&](auto pI) {
          constexpr int p = decltype(pI)::value, PR = S::c[p / S::n], PC = S::c[p % S::n];
          const uint32_t st = it % WS_STAGES;
          ws_bar_wait(&full[st], (it / WS_STAGES) & 1);
          consume_part_reg<K, PR, PC>(sVbuf + st * K::VSTAGE, sU + sig_qoff<SIG>(p) * CC * BN, acc, tm, tn, p == 0);
          __syncwarp();
          if (lane == 0) ws_bar_arrive(&empty[st]);
          ++it;
        });
      }
      // epilogue: 2x2 tiles -> NCHW from the accumulator registers
      bool bad = false;
#pragma unroll
      for (int i = 0; i < TM; ++i) {
        const int tile = tb * BM + tm + 32 * i;
        if (tile >= d.tiles) continue;
        const int tx = tile % d.tw;
        const int t2 = tile / d.tw;
        const int ty = t2 % d.th;
        const int n = t2 / d.th;
#pragma unroll
        for (int jp = 0; jp < NP; ++jp) {
#pragma unroll
          for (int half = 0; half < 2; ++half) {
            const int f = f0 + tn * TN + 2 * jp + half;
            if (f >= F) continue;
            float* yf = y + ((size_t)n * F + f) * (size_t)d.oh * d.ow;
#pragma unroll
            for (int ii = 0; ii < 2; ++ii) {
              const int oy = 2 * ty + ii;
              if (oy >= d.oh) continue;
              const float2 a0 = upk(acc[i][jp][ii][0]);
              const float2 a1 = upk(acc[i][jp][ii][1]);
              const float v0 = half ? a0.y : a0.x, v1 = half ? a1.y : a1.x;
              const int ox = 2 * tx;
              float* dst = yf + (size_t)oy * d.ow + ox;
              if (ox + 1 < d.ow) {
                bad |= !(isfinite(v0) && isfinite(v1));
                if ((d.ow & 1) == 0 && ((uintptr_t)y & 7) == 0) {
                  __stcs(reinterpret_cast<float2*>(dst), make_float2(v0, v1));
                } else {
                  __stcs(dst, v0);
                  __stcs(dst + 1, v1);
                }
              } else {
                bad |= !isfinite(v0);
                __stcs(dst, v0);
              }
            }
          }
        }
      }
      if (bad && flag) *flag = 1;
    }
  }
}

template <class K>
int launch_ws(const dwm_desc_t& d, const float* x, const float* U, float* y, int32_t* flag, cudaStream_t s) {
  const size_t smem = K::smem_bytes(d.num_freqs);
  // plan-specialized kernels for RGB stems only (C_in = 3; compile time)
  static const bool sig_off = getenv("DWM_SMALLC_NOSIG") != nullptr;  // (experiments)
  constexpr bool sig_ok = K::CC == 3;
  const int sig = (sig_off || !sig_ok) ? 0 : match_plan_sig(d);
  const void* kern = (const void*)small_c_ws_kernel<K, 0>;
  if constexpr (sig_ok) {
    if (sig == 1) kern = (const void*)small_c_ws_kernel<K, 1>;
  }
  if (int st = ensure_dynamic_smem(kern, smem)) return st;
  int sms = 0;
  if (int st = device_sm_count(&sms)) return st;
  const int fblocks = (d.f + K::BN - 1) / K::BN;
  const int64_t nblocks = (d.tiles + K::BM - 1) / K::BM;
  int64_t gx = ((int64_t)sms + fblocks - 1) / fblocks;
  if (gx > nblocks) gx = nblocks;
  const dim3 grid((unsigned)gx, (unsigned)fblocks);
  if constexpr (sig_ok) {
    if (sig == 1) small_c_ws_kernel<K, 1><<<grid, WS_THREADS, smem, s>>>(d, x, U, y, flag);
    else small_c_ws_kernel<K, 0><<<grid, WS_THREADS, smem, s>>>(d, x, U, y, flag);
  } else {
    small_c_ws_kernel<K, 0><<<grid, WS_THREADS, smem, s>>>(d, x, U, y, flag);
  }
  DWM_CUDA_TRY(cudaGetLastError());
  return DWM_OK;
}

template <class K>
int launch_cfg(const dwm_desc_t& d, const float* x, const float* U, float* y, int32_t* flag, cudaStream_t s) {
  const size_t smem = K::smem_bytes(d.num_freqs);
  const void* kern = (const void*)small_c_kernel<K>;
  if (int st = ensure_dynamic_smem(kern, smem)) return st;
  int sms = 0, per_sm = 0;
  if (int st = device_sm_count(&sms)) return st;
  if (int st = cached_occupancy(kern, THREADS, smem, &per_sm)) return st;
  if (per_sm < 1) return fail(DWM_EUNSUPPORTED, "small-C kernel does not fit (smem %zu B)", smem);
  const int fblocks = (d.f + K::BN - 1) / K::BN;
  const int64_t nblocks = (d.tiles + K::BM - 1) / K::BM;
  int64_t gx = ((int64_t)sms * per_sm + fblocks - 1) / fblocks;
  if (gx > nblocks) gx = nblocks;
  small_c_kernel<K><<<dim3((unsigned)gx, (unsigned)fblocks), THREADS, smem, s>>>(d, x, U, y, flag);
  DWM_CUDA_TRY(cudaGetLastError());
  return DWM_OK;
}

constexpr size_t SMEM_CAP = 220 * 1024;

// Wide variant (2 tiles x 8 filters per thread, 64x64 block) when its resident
// U fits; else Tall (1 x 8, 32x64 block); else Narrow (4 x 4, 128x32 block).
// (Measured on cfg2/cfg3 against 2x4, 1x4, 1x8 with 2 CTAs/SM: see DESIGN.md.)
template <int CC>
int launch_cc(const dwm_desc_t& d, const float* x, const float* U, float* y, int32_t* flag, cudaStream_t s) {
  // warp-specialized kernel first: 64 tiles x 64 filters when F > 32, 64 x 48
  // for F a multiple of 48 but not of 64, 32 x 64 when U is large
  static const bool ws_off = getenv("DWM_SMALLC_LEGACY") != nullptr;
  if (!ws_off) {
    using W64 = WsCfg<CC, 2, 8>;
    using W48 = WsCfg<CC, 2, 6>;
    using T64 = WsCfg<CC, 1, 8>;
    if (d.f % 64 != 0 && d.f % 48 == 0 && W48::smem_bytes(d.num_freqs) <= SMEM_CAP)
      return launch_ws<W48>(d, x, U, y, flag, s);
    if (d.f > 32 && W64::smem_bytes(d.num_freqs) <= SMEM_CAP) return launch_ws<W64>(d, x, U, y, flag, s);
    if (d.f > 32 && T64::smem_bytes(d.num_freqs) <= SMEM_CAP) return launch_ws<T64>(d, x, U, y, flag, s);
  }
  using Wide = Cfg<CC, 2, 8>;
  using Narrow = Cfg<CC, 4, 4>;
  using Tall = Cfg<CC, 1, 8>;
  using Tall6 = Cfg<CC, 1, 6>;  // 32 tiles x 48 filters: F = 96, 144, ... without a half-empty block
  if (d.f > 32 && Wide::smem_bytes(d.num_freqs) <= SMEM_CAP) return launch_cfg<Wide>(d, x, U, y, flag, s);
  if (d.f % 64 != 0 && d.f % 48 == 0 && Tall6::smem_bytes(d.num_freqs) <= SMEM_CAP)
    return launch_cfg<Tall6>(d, x, U, y, flag, s);
  // many frequencies (e.g. 11x11/4: 225): keep 64 filters per block -- one V
  // transform feeds twice the filters -- with a 32-tile block (cfg3: 1.34x)
  if (d.f > 32 && Tall::smem_bytes(d.num_freqs) <= SMEM_CAP) return launch_cfg<Tall>(d, x, U, y, flag, s);
  return launch_cfg<Narrow>(d, x, U, y, flag, s);
}

}  // namespace smallc
}  // namespace dwm

namespace dwm {
namespace smallc {
extern template int launch_cc<1>(const dwm_desc_t&, const float*, const float*, float*, int32_t*, cudaStream_t);
extern template int launch_cc<2>(const dwm_desc_t&, const float*, const float*, float*, int32_t*, cudaStream_t);
extern template int launch_cc<3>(const dwm_desc_t&, const float*, const float*, float*, int32_t*, cudaStream_t);
extern template int launch_cc<4>(const dwm_desc_t&, const float*, const float*, float*, int32_t*, cudaStream_t);
}  // namespace smallc
}  // namespace dwm
