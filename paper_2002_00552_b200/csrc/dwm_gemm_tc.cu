// dwm_gemm_tc.cu -- transform-domain contraction on the 5th-gen tensor cores
// (tcgen05, kind::tf32, 3xTF32 split) with the output transform, the
// plan-order part sum and the 2x2 tile interleave fused into the epilogue.
//
// Reference rows: M (engines.py:82-89,189) and A/Sigma/F
// (engines.py:192-194, tensor.py:68-81, engines.py:255).
//
// Per frequency q (all parts, plan order), per 128-tile x 64-filter block:
//   M_q[tile][f] = sum_c V_q[tile][c] * U_q[f][c]
// in FP32 from 3 TF32 products: Vhi*Uhi + Vhi*Ulo + Vlo*Uhi, where
// hi = rn_tf32(x), lo = x - hi (the tensor core truncates lo to TF32).
// U_hi/U_lo come pre-split from the filter transform; V is split on the fly.
//
// MMA shape.  The B operand of one stage is [U_hi (64 filters); U_lo (64)]
// (128 rows, one SW128 tile), so per K = 8 slice two MMAs do all three
// products:
//   D[  0.. 63] (+)= V_hi * U_hi^T                 (N = 128, both halves
//   D[ 64..127] (+)= V_hi * U_lo^T                  in one instruction)
//   D[ 64..127]  += V_lo * U_hi^T                  (N = 64)
// i.e. a main accumulator and a correction accumulator side by side.  N = 128
// runs at 1.4x the FLOP rate of N = 64 (tools/tc_probe.cu: 1034 vs 737 TF/s).
//
// Accuracy.  The tcgen05 FP32 accumulator truncates toward zero (~-0.5 ulp
// per MMA, tools/tc_accum_probe.cu), so a long chain is biased.  Both
// accumulators are therefore fresh per chunk of CH channels (64 for C >= 128,
// 32 otherwise); the epilogue forms chunk = main + corr and sums chunks in
// FP32 round-to-nearest (tools/tc_accuracy_emul.py scheme "pair64": MSE 0.35-
// 0.61x the reference DWM32's on cfg4/cfg5).  Then
//   Y_(i,j) += At_r[i][a] * At_c[j][b] * M_q     (coefficients 0, +-1)
// with Y held in the epilogue warps' registers (4 positions x 32 filters per
// thread), and only y = interleave(Y) reaches HBM.
//
// Warp roles (512 threads, one CTA per SM, persistent over work items;
// register budgets redistributed with setmaxnreg per warpgroup):
//   WG0 warps 0-3   converter (64 regs): V rows (one tile per thread) from the
//                   TMA stage -> hi/lo -> tcgen05.st into a TMEM A slot
//   WG1/2 warps 4-11 epilogue (192 regs): tcgen05.ld chunk accumulators ->
//                   M_q -> Y (registers) -> y (NCHW), non-finite flag.  TMEM
//                   lane quadrant = warp % 4, filter half = (warp - 4) / 4.
//   WG3 warp 12     TMA producer (64 regs): V [128 tiles][32 ch] and
//                   U_hi/U_lo [64 f][32 ch] per (frequency, 32-channel) stage
//       warp 13     TMEM allocator + MMA issuer (elect.sync from the converged warp)
//       warps 14-15 idle (warpgroup padding for setmaxnreg)
// TMEM columns: accumulators 2 x 128 (0-255: main | corr), A slots 4 x 64
// (256-511: V_hi 32 | V_lo 32).
#include <cuda.h>
#include <unistd.h>
#include <cstdlib>
#include <cstdio>
#include <cudaTypedefs.h>

#include "dwm_common.cuh"
#include "dwm_kernels.h"
#include "dwm_sm100.cuh"

namespace dwm {
namespace {

using namespace sm100;

constexpr int BM = 128;        // tiles per work item (MMA M, TMEM lanes)
constexpr int BN = 64;         // filters per work item
constexpr int BK = 32;         // channels per SW128 atom (128 B rows)
constexpr int SK = 64;         // channels per pipeline stage (2 atoms)
constexpr int STAGES = 3;      // smem ring: 3 x (V 32 KB + U 32 KB)
constexpr int A_SLOTS = 2;     // TMEM A ring: 2 x (hi 64 | lo 64) columns
#ifndef DWM_TC_VPF
#define DWM_TC_VPF 4
#endif
constexpr int V_PREFETCH = DWM_TC_VPF;  // stages of V prefetched into L2 ahead of the TMA loads
constexpr int THREADS = 512;
constexpr int EPI_WARPS = 8;
constexpr int EC = 32;         // filter columns per epilogue warp
constexpr int WARP_TMA = 12, WARP_MMA = 13;
constexpr int MAX_FREQS = 1024;
constexpr uint32_t ATOM_BYTES = BM * BK * 4;  // 16 KB: one [128 rows][32 ch] SW128 tile
constexpr uint32_t COL_ACC = 0, COL_A = 256;
constexpr int REG_CONV = 72, REG_EPI = 192, REG_CTRL = 56;
static_assert(4 * 32 * (REG_CONV + REG_CTRL) + 8 * 32 * REG_EPI <= 65536, "register file");

struct __align__(1024) Smem {
  float v[STAGES][2][BM * BK];      // [stage][atom][128 tiles][32 ch]
  float u[STAGES][2][2 * BN * BK];  // [stage][atom][U_hi 64 rows; U_lo 64 rows][32 ch]
  uint64_t b_full[STAGES];          // TMA -> converter (V) and MMA (U)
  uint64_t done[STAGES];            // MMA commit per stage -> TMA, converter, epilogue
  uint64_t a_full[A_SLOTS];         // converter -> MMA
  uint64_t acc_empty[2];            // epilogue -> MMA
  uint32_t tmem_base;
  int8_t coef[MAX_FREQS][4];
};

__device__ __forceinline__ int at_coef_rt(int r, int i, int a) {
  return r == 1 ? (i == a ? 1 : 0)
       : r == 2 ? (i == 0 ? (a <= 1 ? 1 : 0) : (a == 1 ? 1 : (a == 2 ? -1 : 0)))
                : (i == 0 ? (a <= 2 ? 1 : 0) : (a == 0 ? 0 : (a == 1 ? 1 : -1)));
}

// Profiling builds (-DDWM_TC_PROFILE, tools/tc_profile.py): per-role cycles
// spent in mbarrier waits and in total, summed over CTAs, plus timing-only
// ablation switches (g_tc_flags; results are wrong when any is set):
//   1 converter does no V reads / TMEM stores   2 epilogue does no TMEM loads
//   4 no V_lo * U_hi MMA                        8 TMA loads U only
#ifdef DWM_TC_PROFILE
__device__ unsigned long long g_tc_prof[32];
__device__ int g_tc_flags;
#define PWAIT(slot, bar, ph) do { const long long _t = clock64(); mbar_wait(bar, ph); prof[slot] += clock64() - _t; } while (0)
#define PFLAG(b) (g_tc_flags & (b))
#else
#define PWAIT(slot, bar, ph) mbar_wait(bar, ph)
#define PFLAG(b) 0
#endif

template <uint32_t N>
__device__ __forceinline__ void setmaxnreg_inc() { asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(N)); }
template <uint32_t N>
__device__ __forceinline__ void setmaxnreg_dec() { asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(N)); }

// The tcgen05 FP32 accumulator truncates each K = 8 step toward zero (about
// -0.5 ulp per step, tools/tc_accum_probe.cu), so a chunk of n main-product
// steps is biased toward zero by ~n/2 ulp of its value.  For the 32-channel
// chunks (4 steps, C < 128, where the GEMM error weighs most) the epilogue
// adds back 1 ulp away from zero -- one integer add on the float's bits (a
// mantissa carry into the exponent is still +1 ulp) -- emulated MSE 0.56-0.70x
// the reference DWM32's instead of 0.70-0.86x (tools/tc_accuracy_emul.py
// "pairc32_25").  The 64-channel chunks do not use it: on the C >= 128
// shapes the extra epilogue latency cost 4-8 % (profiles/r2/ab_tc_bias_comp_chunk128.txt)
// and their MSE is already 0.2-0.55x.
__device__ __forceinline__ float trunc_compensate(float x, uint32_t k) {
  return __uint_as_float(__float_as_uint(x) + k);
}

// Stage geometry: stage kc of a frequency covers channels [64 kc, 64 kc + 64);
// a C % 64 == 32 tail stage has one atom (4 K-slices).
__device__ __forceinline__ int stage_atoms(int C, int kc) { return C - SK * kc >= SK ? 2 : 1; }

// C32: 32-channel accumulator chunks (C < 128) with the truncation-bias
// compensation; otherwise 64-channel chunks, uncompensated.
template <bool C32>
__global__ void __launch_bounds__(THREADS, 1)
gemm_tc_kernel(const dwm_desc_t d, const __grid_constant__ CUtensorMap map_v, const __grid_constant__ CUtensorMap map_u,
               float* __restrict__ y, int32_t* __restrict__ flag) {
  constexpr bool chunk32 = C32;
  extern __shared__ uint8_t smem_raw[];
  Smem& S = *reinterpret_cast<Smem*>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const int Q = d.num_freqs, F = d.f, C = d.c;
  const int KS = (C + SK - 1) / SK;        // stages per frequency
  const int n_nblk = (F + BN - 1) / BN;    // a partial last block computes zero columns, never stored
  const int64_t n_mblk = (d.tiles + BM - 1) / BM;
  const int64_t n_items = n_mblk * n_nblk;

  // ---- one-time setup
  if (tid == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&S.b_full[i], 1);
      mbar_init(&S.done[i], 1);
    }
    for (int i = 0; i < A_SLOTS; ++i) mbar_init(&S.a_full[i], 4);
    for (int i = 0; i < 2; ++i) mbar_init(&S.acc_empty[i], EPI_WARPS);
    fence_barrier_init();
  }
  // output-transform coefficient of every frequency for the 4 tile positions
  for (int q = tid; q < Q; q += THREADS) {
    int rem = q, pr = 0, pc = 0, a = 0, b = 0;
    for (int rp = 0, found = 0; rp < d.n_row_parts && !found; ++rp)
      for (int cp = 0; cp < d.n_col_parts; ++cp) {
        const int cr = d.row_parts[rp].count, cc = d.col_parts[cp].count;
        const int nq = (cr + 1) * (cc + 1);
        if (rem < nq) { pr = cr; pc = cc; a = rem / (cc + 1); b = rem % (cc + 1); found = 1; break; }
        rem -= nq;
      }
    for (int i = 0; i < 2; ++i)
      for (int j = 0; j < 2; ++j) S.coef[q][i * 2 + j] = (int8_t)(at_coef_rt(pr, i, a) * at_coef_rt(pc, j, b));
  }
  if (warp == WARP_TMA && lane == 0) {
    tma_prefetch_desc(&map_v);
    tma_prefetch_desc(&map_u);
  }
  if (warp == WARP_MMA) tmem_alloc<512>(&S.tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = S.tmem_base;
#ifdef DWM_TC_PROFILE
  long long prof[4] = {0, 0, 0, 0};
  const long long t_start = clock64();
#endif

  if (warp >= 12) {
    setmaxnreg_dec<REG_CTRL>();
    if (warp == WARP_TMA) {
      // ================= TMA producer (whole warp converged, one lane issues) =================
      uint32_t it = 0;
      for (int64_t w = blockIdx.x; w < n_items; w += gridDim.x) {
        const int blk = (int)(w % n_nblk);
        const int m0 = (int)(w / n_nblk) * BM;
        for (int q = 0; q < Q; ++q)
          for (int kc = 0; kc < KS; ++kc, ++it) {
            const uint32_t s = it % STAGES;
            if (it >= STAGES) PWAIT(0, &S.done[s], ((it - STAGES) / STAGES) & 1);
            if (elect_one()) {
              const int na = stage_atoms(C, kc);
              mbar_arrive_expect_tx(&S.b_full[s], na * ((PFLAG(8) ? 0 : ATOM_BYTES) + ATOM_BYTES));
              const int urow = (q * n_nblk + blk) * (2 * BN);
              for (int h = 0; h < na; ++h) {
                if (!PFLAG(8)) tma_load_3d(S.v[s][h], &map_v, &S.b_full[s], SK * kc + BK * h, m0, q);
                tma_load_2d(S.u[s][h], &map_u, &S.b_full[s], SK * kc + BK * h, urow);
              }
              // V comes from HBM (the input transform just wrote it; the 3
              // smem stages hide ~3 us less than its latency under load):
              // prefetch the V box of stage it + V_PREFETCH into L2
              if (V_PREFETCH > 0 && !PFLAG(8)) {
                int nq = q, nk = kc + V_PREFETCH, nm = m0;
                nq += nk / KS;
                nk %= KS;
                if (nq >= Q) {
                  nq -= Q;
                  nm = (int)((w + gridDim.x) / n_nblk) * BM;
                }
                if (nm < d.tiles && nq < Q)
                  for (int h = 0; h < stage_atoms(C, nk); ++h) tma_prefetch_3d(&map_v, SK * nk + BK * h, nm, nq);
              }
            }
            __syncwarp();
          }
      }
    } else if (warp == WARP_MMA) {
      // ================= MMA issuer (whole warp converged, one lane issues) =================
      // one tcgen05.commit per 64-channel stage: each commit costs the tensor
      // pipe a ~140-cycle bubble (tools/commit_probe.cu), so the stage is the
      // unit of every release (smem stage, A slot, accumulator chunk)
      const uint32_t idesc128 = idesc_tf32(BM, 2 * BN), idesc64 = idesc_tf32(BM, BN);
      uint32_t it = 0, uses0 = 0, uses1 = 0, st2 = 0;
      for (int64_t w = blockIdx.x; w < n_items; w += gridDim.x) {
        for (int q = 0; q < Q; ++q) {
          for (int kc = 0; kc < KS; ++kc, ++it) {
            const uint32_t sb = it % STAGES, sa = it % A_SLOTS;
            const int na = stage_atoms(C, kc);
            // accumulator buffers of this stage: chunk32 == 0 -> one 64-channel
            // chunk in buffer (st2 % 2); chunk32 == 1 -> two 32-channel chunks,
            // buffers 0 and 1
            const uint32_t b0 = chunk32 ? 0u : (st2 & 1u);
            const bool use0 = chunk32 || b0 == 0, use1 = chunk32 ? na == 2 : b0 == 1;
            if (use0) { PWAIT(0, &S.acc_empty[0], (uses0 & 1) ^ 1); ++uses0; }
            if (use1) { PWAIT(0, &S.acc_empty[1], (uses1 & 1) ^ 1); ++uses1; }
            // no b_full wait: the converter signals a_full only after it
            // observed b_full, and the same TMA transaction carried U
            PWAIT(1, &S.a_full[sa], (it / A_SLOTS) & 1);
            tc_fence_after();
            const uint32_t a_hi = tmem + COL_A + sa * (4 * BK), a_lo = a_hi + 2 * BK;
            if (elect_one()) {
              for (int h = 0; h < na; ++h) {
                const uint64_t du = sdesc_sw128(smem_u32(S.u[sb][h]));
                const uint32_t buf = chunk32 ? (uint32_t)h : b0;
                const uint32_t dacc = tmem + COL_ACC + buf * (2 * BN);
#pragma unroll
                for (int k = 0; k < BK / 8; ++k) {
                  // +32 B per K = 8 slice, in 16-byte descriptor units
                  const bool fresh = k == 0 && (chunk32 || h == 0);
                  mma_tf32_ts(dacc, a_hi + BK * h + 8 * k, du + 2 * k, idesc128, fresh ? 0u : 1u);
                  if (!PFLAG(4)) mma_tf32_ts(dacc + BN, a_lo + BK * h + 8 * k, du + 2 * k, idesc64, 1u);
                }
              }
              mma_commit(&S.done[sb]);
            }
            __syncwarp();
            ++st2;
          }
        }
      }
    }
  } else if (warp < 4) {
    setmaxnreg_dec<REG_CONV>();
    // ================= converter: V stage (smem) -> hi/lo -> TMEM A slot =================
    const uint32_t lane_addr = tmem + ((uint32_t)(32 * warp) << 16);
    const int m = 32 * warp + lane;
    uint32_t it = 0;
    for (int64_t w = blockIdx.x; w < n_items; w += gridDim.x) {
      for (int q = 0; q < Q; ++q) {
        for (int kc = 0; kc < KS; ++kc, ++it) {
          const uint32_t sb = it % STAGES, sa = it % A_SLOTS;
          const int na = stage_atoms(C, kc);
          PWAIT(0, &S.b_full[sb], (it / STAGES) & 1);
          // A slot sa was last read by the MMAs of stage it - 2
          if (it >= A_SLOTS) PWAIT(1, &S.done[(it - A_SLOTS) % STAGES], ((it - A_SLOTS) / STAGES) & 1);
          tc_fence_after();
          const uint32_t base = lane_addr + COL_A + sa * (4 * BK);
          for (int h = 0; h < na; ++h) {
            if (PFLAG(1)) break;
            const uint8_t* vrow = reinterpret_cast<const uint8_t*>(S.v[sb][h]);
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
              float hi[16], lo[16];
#pragma unroll
              for (int c4 = 0; c4 < 4; ++c4) {
                // row m, 16-byte chunk (4 hh + c4) of the SWIZZLE_128B tile
                const float4 x = *reinterpret_cast<const float4*>(vrow + sw128_offset(m, 16 * hh + 4 * c4));
                const float xs[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  // hi = tf32 round-to-nearest (ties away) in 2 integer ops; lo = x - hi
                  // exactly, handed to the tensor core raw (it truncates lo to tf32)
                  const float hv = __uint_as_float((__float_as_uint(xs[e]) + 0x1000u) & 0xFFFFE000u);
                  hi[c4 * 4 + e] = hv;
                  lo[c4 * 4 + e] = __fsub_rn(xs[e], hv);
                }
              }
              tmem_st16(base + BK * h + 16 * hh, hi);
              tmem_st16(base + 2 * BK + BK * h + 16 * hh, lo);
            }
          }
          tmem_st_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&S.a_full[sa]);
        }
      }
    }
  } else {
    setmaxnreg_inc<REG_EPI>();
    // ================= epilogue: chunks -> M_q -> Y (registers) -> y =================
    const int quad = warp % 4;
    const int c0 = ((warp - 4) / 4) * EC;
    const uint32_t lane_addr = tmem + ((uint32_t)(32 * quad) << 16);
    const int m = 32 * quad + lane;
    uint32_t it = 0, st2 = 0;
    for (int64_t w = blockIdx.x; w < n_items; w += gridDim.x) {
      const int64_t tile = (w / n_nblk) * BM + m;
      const int n0 = (int)(w % n_nblk) * BN;
      float Y[4][EC];
#pragma unroll
      for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int j = 0; j < EC; ++j) Y[p][j] = 0.f;
      for (int q = 0; q < Q; ++q) {
        float mq[EC];
        for (int kc = 0; kc < KS; ++kc, ++it, ++st2) {
          const int na = stage_atoms(C, kc);
          PWAIT(0, &S.done[it % STAGES], (it / STAGES) & 1);
          tc_fence_after();
          const int nb = chunk32 ? na : 1;
          for (int bi = 0; bi < nb; ++bi) {
            const uint32_t buf = chunk32 ? (uint32_t)bi : (st2 & 1u);
            const bool first = kc == 0 && bi == 0;
            const uint32_t acc = lane_addr + COL_ACC + buf * (2 * BN) + c0;
#pragma unroll
            for (int h = 0; h < EC / 8; ++h) {
              if (PFLAG(2)) { mq[8 * h] = 0.f; continue; }
              float mn[8], cr[8];
              tmem_ld8(acc + 8 * h, mn);
              tmem_ld8(acc + BN + 8 * h, cr);
              tmem_ld_wait();
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                const float part = __fadd_rn(chunk32 ? trunc_compensate(mn[j], 1u) : mn[j], cr[j]);
                mq[8 * h + j] = first ? part : __fadd_rn(mq[8 * h + j], part);
              }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&S.acc_empty[buf]);
          }
        }
        // output transform: Y_p +-= M_q for the positions p with a nonzero coefficient
        const char4 cf = *reinterpret_cast<const char4*>(S.coef[q]);
        const int8_t cfa[4] = {cf.x, cf.y, cf.z, cf.w};
#pragma unroll
        for (int p = 0; p < 4; ++p) {
          if (cfa[p] > 0) {
#pragma unroll
            for (int j = 0; j < EC; ++j) Y[p][j] = __fadd_rn(Y[p][j], mq[j]);
          } else if (cfa[p] < 0) {
#pragma unroll
            for (int j = 0; j < EC; ++j) Y[p][j] = __fsub_rn(Y[p][j], mq[j]);
          }
        }
      }
      // Y -> y: positions (i, j) of tile (n, ty, tx), this warp's filters
      if (tile < d.tiles) {
        const int tx = (int)(tile % d.tw);
        const int64_t t2 = tile / d.tw;
        const int ty = (int)(t2 % d.th);
        const int n = (int)(t2 / d.th);
        const int oy = 2 * ty, ox = 2 * tx;
        const bool pair = ox + 1 < d.ow, vec = pair && (d.ow & 1) == 0 && ((uintptr_t)y & 7) == 0;
        bool bad = false;
#pragma unroll
        for (int j = 0; j < EC; ++j) {
          const int f = n0 + c0 + j;
          if (f >= F) break;
          float* yf = y + ((size_t)n * F + f) * (size_t)d.oh * d.ow + (size_t)oy * d.ow + ox;
#pragma unroll
          for (int ii = 0; ii < 2; ++ii) {
            if (oy + ii >= d.oh) continue;
            const float v0 = Y[2 * ii][j], v1 = Y[2 * ii + 1][j];
            float* dst = yf + ii * d.ow;
            if (vec) {
              bad |= !(isfinite(v0) && isfinite(v1));
              __stcs(reinterpret_cast<float2*>(dst), make_float2(v0, v1));
            } else {
              bad |= !isfinite(v0);
              __stcs(dst, v0);
              if (pair) {
                bad |= !isfinite(v1);
                __stcs(dst + 1, v1);
              }
            }
          }
        }
        if (bad && flag) *flag = 1;
      }
    }
  }

#ifdef DWM_TC_PROFILE
  {
    // role r: 0 TMA (warp 12), 1 MMA (warp 13), 2 converter (warp 0), 3 epilogue (warp 4)
    const int role = warp == WARP_TMA ? 0 : warp == WARP_MMA ? 1 : warp == 0 ? 2 : warp == 4 ? 3 : -1;
    if (role >= 0 && lane == 0) {
      atomicAdd(&g_tc_prof[role * 4 + 0], (unsigned long long)prof[0]);
      atomicAdd(&g_tc_prof[role * 4 + 1], (unsigned long long)prof[1]);
      atomicAdd(&g_tc_prof[role * 4 + 3], (unsigned long long)(clock64() - t_start));
    }
  }
#endif
  tc_fence_before();
  __syncthreads();
  if (warp == WARP_MMA) tmem_dealloc<512>(tmem);
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
  }
  return fn;
}

int make_v_map(CUtensorMap* map, const float* base, const dwm_desc_t& d) {
  auto encode = get_encode();
  if (!encode) return fail(DWM_ECUDA, "cuTensorMapEncodeTiled is unavailable");
  // [freq][tiles][C]: rows past `tiles` of a frequency read as zeros
  const cuuint64_t dims[3] = {(cuuint64_t)d.c, (cuuint64_t)d.tiles, (cuuint64_t)d.num_freqs};
  const cuuint64_t strides[2] = {(cuuint64_t)d.c * sizeof(float), (cuuint64_t)d.tiles * d.c * sizeof(float)};
  const cuuint32_t box[3] = {BK, BM, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, (void*)base, dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(DWM_ECUDA, "cuTensorMapEncodeTiled(V) failed (%d)", (int)r);
  return DWM_OK;
}

// U in the stacked tcgen05 layout: [freq][64-filter block][U_hi 64 rows; U_lo 64 rows][C]
int make_u_map(CUtensorMap* map, const float* base, const dwm_desc_t& d) {
  auto encode = get_encode();
  if (!encode) return fail(DWM_ECUDA, "cuTensorMapEncodeTiled is unavailable");
  const int64_t nblk = (d.f + BN - 1) / BN;
  const cuuint64_t dims[2] = {(cuuint64_t)d.c, (cuuint64_t)(d.num_freqs * nblk * 2 * BN)};
  const cuuint64_t strides[1] = {(cuuint64_t)d.c * sizeof(float)};
  const cuuint32_t box[2] = {BK, 2 * BN};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)base, dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(DWM_ECUDA, "cuTensorMapEncodeTiled(U) failed (%d)", (int)r);
  return DWM_OK;
}

}  // namespace

bool tc_gemm_supported(const dwm_desc_t& d) {
  return d.c % BK == 0 && d.f >= 1 && d.num_freqs <= MAX_FREQS && d.tiles < ((int64_t)1 << 31);
}

size_t tc_filter_bytes(const dwm_desc_t& d) {
  return (size_t)d.num_freqs * (size_t)((d.f + BN - 1) / BN) * 2 * BN * (size_t)d.c * sizeof(float);
}

// Accumulator chunk: one 64-channel stage when C >= 128 (emulated MSE
// 0.35-0.61x the reference DWM32's, tools/tc_accuracy_emul.py "pair64"), two
// 32-channel chunks per stage otherwise (C = 64: "pair64" would be one chain
// over all of K, 1.1-1.3x).  DWM_TC_CHUNK=32|64 overrides (experiments).
static int tc_chunk32(const dwm_desc_t& d) {
  static const int env = [] {
    const char* e = getenv("DWM_TC_CHUNK");
    return e ? atoi(e) : 0;
  }();
  if (env == 32) return 1;
  if (env == 64) return 0;
  return d.c >= 128 ? 0 : 1;
}

int launch_gemm_tc(const dwm_desc_t& d, const void* V, const void* U, void* y, int32_t* flag, cudaStream_t s) {
  if (!tc_gemm_supported(d)) return fail(DWM_EUNSUPPORTED, "tcgen05 GEMM needs C %% 32 == 0");
  CUtensorMap mv, mu;
  if (int st = make_v_map(&mv, (const float*)V, d)) return st;
  if (int st = make_u_map(&mu, (const float*)U, d)) return st;
  const size_t smem = sizeof(Smem) + 1024;
  int sms = 0;
  if (int st = device_sm_count(&sms)) return st;
  const int64_t items = ((d.tiles + BM - 1) / BM) * ((d.f + BN - 1) / BN);
  const int grid = (int)(items < sms ? items : sms);
  if (tc_chunk32(d)) {
    if (int st = ensure_dynamic_smem((const void*)gemm_tc_kernel<true>, smem)) return st;
    gemm_tc_kernel<true><<<grid, THREADS, smem, s>>>(d, mv, mu, (float*)y, flag);
  } else {
    if (int st = ensure_dynamic_smem((const void*)gemm_tc_kernel<false>, smem)) return st;
    gemm_tc_kernel<false><<<grid, THREADS, smem, s>>>(d, mv, mu, (float*)y, flag);
  }
  DWM_CUDA_TRY(cudaGetLastError());
  return DWM_OK;
}

}  // namespace dwm

#ifdef DWM_TC_PROFILE
extern "C" int dwm_debug_tc_profile(unsigned long long* out, int reset) {
  cudaDeviceSynchronize();
  if (cudaMemcpyFromSymbol(out, dwm::g_tc_prof, sizeof(unsigned long long) * 32) != cudaSuccess) return 1;
  if (reset) {
    unsigned long long z[32] = {0};
    cudaMemcpyToSymbol(dwm::g_tc_prof, z, sizeof(z));
  }
  return 0;
}
extern "C" int dwm_debug_tc_flags(int flags) {
  return cudaMemcpyToSymbol(dwm::g_tc_flags, &flags, sizeof(int)) == cudaSuccess ? 0 : 1;
}
#endif
