// dwm_gemm_tc.cu -- transform-domain contraction on the 5th-gen tensor cores
// (tcgen05 kind::f16, 3-term fp16 split, fp32 accumulate) with the output
// transform, the plan-order part sum and the 2x2 tile interleave fused into
// the epilogue.
//
// Reference rows: M (engines.py:82-89,189) and A/Sigma/F
// (engines.py:192-194, tensor.py:68-81, engines.py:255).
//
// Per frequency q (all parts, plan order), per 128-tile x 64-filter block:
//   M_q[tile][f] = sum_c V_q[tile][c] * U_q[f][c]
// in FP32 from 3 fp16 products of power-of-two scaled operands:
//   V' = s_v V, U'_f = s_f U_f,  x' = hi + lo (hi = rn_f16(x'), lo = rn_f16(x' - hi))
//   M' = V'hi U'hi + V'hi U'lo + V'lo U'hi,    M = M' / (s_v s_f)
// A 22-bit split like 3xTF32, at the fp16 tensor rate (kind::f16 TS MMAs
// stream 1.68x faster than kind::tf32 for the same N: tools/f16_probe.cu).
// The scales are exact powers of two picked from range bounds, so V' and U'
// sit in [2^12, 2^15) at their maxima: no fp16 overflow, and lo stays normal
// down to 2^-26 of the maximum (MSE is absolute, so smaller values cost
// nothing measurable):
//   s_v = 2^(12 - floor(log2 max|x_n|)) per image n (|V| <= 4 max|x|: Bt rows
//                                       have |.|-sums <= 2); max|x_n| from the
//                                       input transform's staging loads
//                                       (atomicMax per image), so an image's
//                                       bits never depend on its batch-mates
//   s_f = 2^(12 - floor(log2 max|w_f|)) |U_f| <= 2.25 max|w_f| (G: sums <= 1.5)
// U'hi/U'lo come pre-split from the filter transform; V is scaled and split
// on the fly by the converter warps.
//
// MMA shape.  The B operand of one 64-channel stage is [U'hi (64 filters);
// U'lo (64)] (128 rows x 64 fp16 = one SW128 tile), so per K = 16 slice two
// MMAs do all three products:
//   D[  0.. 63] (+)= V'hi * U'hi^T                 (N = 128, both halves
//   D[ 64..127] (+)= V'hi * U'lo^T                  in one instruction)
//   D[ 64..127]  += V'lo * U'hi^T                  (N = 64)
// i.e. a main accumulator and a correction accumulator side by side.
//
// Accuracy.  The tcgen05 FP32 accumulator truncates each MMA step toward zero
// (tools/tc_accum_probe.cu, tools/f16_probe.cu), so both accumulators are
// fresh per chunk of 128 channels (8 K = 16 steps; 64 channels = 4 steps when
// C < 128, with a +1 ulp truncation-bias compensation); the epilogue forms
// chunk = main + corr and sums chunks in FP32 round-to-nearest.  Then
//   Y_(i,j) += At_r[i][a] * At_c[j][b] * M'_q     (coefficients 0, +-1)
// with Y held in the epilogue warps' registers (4 positions x 32 filters per
// thread), y = interleave(Y) / (s_v s_f) is the only HBM write.
//
// Warp roles (512 threads, one CTA per SM, persistent over work items;
// register budgets redistributed with setmaxnreg per warpgroup):
//   WG0 warps 0-3   converter (72 regs): V rows (one tile per thread) from the
//                   TMA stage -> scale -> hi/lo fp16 pairs -> tcgen05.st
//   WG1/2 warps 4-11 epilogue (192 regs): tcgen05.ld chunk accumulators ->
//                   M'_q -> Y (registers) -> y (NCHW), non-finite flag.  TMEM
//                   lane quadrant = warp % 4, filter half = (warp - 4) / 4.
//   WG3 warp 12     V TMA producer (56 regs): V [128 tiles][2 x 32 ch] fp32 per
//                   (frequency, 64-channel) stage into the V ring, which the
//                   converter frees as soon as it has read a stage
//       warp 13     TMEM allocator + MMA issuer (elect.sync from the converged warp)
//       warp 14     U TMA producer: [U'hi; U'lo] [128 rows][64 ch] fp16 per
//                   stage into the U ring, freed by the stage's MMA commit
//       warp 15     idle (warpgroup padding for setmaxnreg)
// TMEM columns: accumulators 2 x 128 (0-255: main | corr), A slots 4 x 64
// (256-511: V'hi 32 | V'lo 32, two fp16 channels per column).
#include <cuda.h>
#include <cuda_fp16.h>
#include <unistd.h>
#include <cstdlib>
#include <cstdio>
#include <cudaTypedefs.h>

#include "dwm_common.cuh"
#include "dwm_filter.cuh"
#include "dwm_kernels.h"
#include "dwm_sm100.cuh"

namespace dwm {
namespace {

using namespace sm100;

constexpr int BM = 128;        // tiles per work item (MMA M, TMEM lanes)
constexpr int BN = 64;         // filters per work item
constexpr int VK = 32;         // fp32 V channels per SW128 atom (128 B rows)
constexpr int SK = 64;         // channels per pipeline stage (2 V atoms, 1 U atom)
#ifndef DWM_TC_VSTAGES
#define DWM_TC_VSTAGES 4
#endif
constexpr int VSTAGES = DWM_TC_VSTAGES;  // V ring: 32 KB stages, freed by the converter
#ifndef DWM_TC_USTAGES
#define DWM_TC_USTAGES 4
#endif
constexpr int USTAGES = DWM_TC_USTAGES;  // U ring (16 KB stages), freed by the MMAs
constexpr int STAGES = 4;      // commit ring (done[]), one commit per stage; = A_SLOTS
constexpr int A_SLOTS = 4;     // TMEM A ring: 4 x (hi 32 | lo 32) columns
#ifndef DWM_TC_U_EVICT_LAST
#define DWM_TC_U_EVICT_LAST 0
#endif
#ifndef DWM_TC_VPF
#define DWM_TC_VPF 4
#endif
constexpr int V_PREFETCH = DWM_TC_VPF;  // stages of V prefetched into L2 ahead of the TMA loads
#ifndef DWM_TC_CONV_WARPS
#define DWM_TC_CONV_WARPS 4
#endif
// 4: one 64-channel row per thread; 8: one 32-channel atom (measured no faster:
// the converter stays ~75 % busy with twice the warps, and the epilogue then
// gets 184 registers and spills -- profiles/r2/ab_tc_conv8.txt)
constexpr int CONV_WARPS = DWM_TC_CONV_WARPS;
constexpr int EPI_WARPS = 8;
constexpr int EPI_WARP0 = CONV_WARPS;
constexpr int THREADS = 32 * (CONV_WARPS + EPI_WARPS + 4);
constexpr int EC = 32;         // filter columns per epilogue warp
constexpr int WARP_TMA = CONV_WARPS + EPI_WARPS, WARP_MMA = WARP_TMA + 1, WARP_UTMA = WARP_TMA + 2;
constexpr int MAX_FREQS = 1024;
constexpr uint32_t V_ATOM_BYTES = BM * VK * 4;   // 16 KB: [128 rows][32 fp32 ch]
constexpr uint32_t U_ATOM_BYTES = 2 * BN * SK * 2;  // 16 KB: [128 rows][64 fp16 ch]
constexpr uint32_t COL_ACC = 0, COL_A = 256, A_COLS = 64;
// setmaxnreg moves registers within the CTA's launch allocation (THREADS x the
// compiled count: 128 at 512 threads, 96 at 640), so the budgets must fit it
constexpr int REG_CONV = CONV_WARPS == 8 ? 40 : 80, REG_EPI = CONV_WARPS == 8 ? 184 : 192,
              REG_CTRL = CONV_WARPS == 8 ? 32 : 48;
constexpr int REG_LAUNCH = CONV_WARPS == 8 ? 96 : 128;
static_assert(32 * (CONV_WARPS * REG_CONV + 4 * REG_CTRL + EPI_WARPS * REG_EPI) <= THREADS * REG_LAUNCH,
              "register budgets exceed the launch allocation");

struct __align__(1024) Smem {
  float v[VSTAGES][2][BM * VK];     // [stage][atom][128 tiles][32 ch] fp32
  uint16_t u[USTAGES][2 * BN * SK];  // [stage][U'hi 64 rows; U'lo 64 rows][64 ch] fp16
  uint64_t v_full[VSTAGES];         // V TMA -> converter
  uint64_t v_empty[VSTAGES];        // converter (V read) -> V TMA
  uint64_t u_full[USTAGES];         // U TMA -> MMA
  uint64_t done[STAGES];            // MMA commit per stage -> U TMA, converter, epilogue
  uint64_t a_full[A_SLOTS];         // converter -> MMA
  uint64_t acc_empty[2];            // epilogue -> MMA
  uint32_t tmem_base;
  uint8_t coef[MAX_FREQS];           // output-transform sign of the 4 tile positions, 2 bits each
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

// The tcgen05 FP32 accumulator truncates each MMA step toward zero, so a
// chunk of n steps is biased toward zero by ~n/2 ulp of its value.  For the
// 64-channel chunks (4 K = 16 steps, C < 128, where the GEMM error weighs
// most) the epilogue adds back 1 ulp away from zero -- one integer add on the
// float's bits (a mantissa carry into the exponent is still +1 ulp).
__device__ __forceinline__ float trunc_compensate(float x, uint32_t k) {
  return __uint_as_float(__float_as_uint(x) + k);
}

// x - hi for a pair (hi = the f16x2 rounding of x), exact in fp32: two
// mixed-precision FMAs (FHFMA, f16 operand from a register half) instead of
// unpacking hi to fp32 first.
__device__ __forceinline__ float2 residual_f16x2(uint32_t hi, float2 x) {
  float2 r;
  asm("{\n\t.reg .f16 a, b, m1;\n\tmov.b32 {a, b}, %2;\n\tmov.b16 m1, 0xBC00;\n\t"
      "fma.rn.f32.f16 %0, a, m1, %3;\n\tfma.rn.f32.f16 %1, b, m1, %4;\n\t}"
      : "=f"(r.x), "=f"(r.y)
      : "r"(hi), "f"(x.x), "f"(x.y));
  return r;
}

// Power-of-two operand scale from the bits of a max |value| (floor(log2) = e):
// s = 2^(12 - e), clamped to normal floats; 0 -> 1; inf/nan -> tiny (the
// non-finite values propagate to y and the flag).
__host__ __device__ __forceinline__ int scale_exp(uint32_t maxbits) {
  const int e = (int)((maxbits >> 23) & 0xFF) - 127;  // exponent field (subnormal/0: -127)
  if (maxbits == 0) return 0;
  const int k = 12 - e;
  return k > 126 ? 126 : (k < -126 ? -126 : k);
}
__device__ __forceinline__ float exp2i(int k) { return __uint_as_float((uint32_t)(127 + k) << 23); }

// Stage geometry: stage kc of a frequency covers channels [64 kc, 64 kc + 64);
// a C % 64 == 32 tail stage has one V atom (2 K = 16 slices).
__device__ __forceinline__ int stage_atoms(int C, int kc) { return C - SK * kc >= SK ? 2 : 1; }

// CHS: stages per accumulator chunk (2: 128 channels, 1: 64 channels + compensation)
template <int CHS>
__global__ void __launch_bounds__(THREADS, 1)
gemm_tc_kernel(const dwm_desc_t d, const __grid_constant__ CUtensorMap map_v, const __grid_constant__ CUtensorMap map_u,
               const float* __restrict__ inv_f, const uint32_t* __restrict__ xmax_slots, float* __restrict__ y,
               int32_t* __restrict__ flag, int pf_all) {
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
    for (int i = 0; i < VSTAGES; ++i) {
      mbar_init(&S.v_full[i], 1);
      mbar_init(&S.v_empty[i], CONV_WARPS);
    }
    for (int i = 0; i < USTAGES; ++i) mbar_init(&S.u_full[i], 1);
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&S.done[i], 1);
    }
    for (int i = 0; i < A_SLOTS; ++i) mbar_init(&S.a_full[i], CONV_WARPS);
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
    uint32_t code = 0;  // 2 bits per position p = 2 i + j: 0 -> 0, 1 -> +1, 3 -> -1
    for (int i = 0; i < 2; ++i)
      for (int j = 0; j < 2; ++j) code |= ((uint32_t)(at_coef_rt(pr, i, a) * at_coef_rt(pc, j, b)) & 3u) << (2 * (2 * i + j));
    S.coef[q] = (uint8_t)code;
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
  // per-image V scale exponent of tile row m of work item w (rows past the
  // last tile take the last image's; they are computed but never stored)
  const int64_t tiles_img = (int64_t)d.th * d.tw;
  auto row_scale_exp = [&](int64_t w, int m) {
    const int64_t t = min((w / n_nblk) * BM + m, d.tiles - 1);
    return scale_exp(__ldg(xmax_slots + t / tiles_img));
  };
#ifdef DWM_TC_PROFILE
  long long prof[4] = {0, 0, 0, 0};
  const long long t_start = clock64();
#endif

  if (warp >= WARP_TMA) {
    setmaxnreg_dec<REG_CTRL>();
    if (warp == WARP_TMA) {
      // ================= V TMA producer (whole warp converged, one lane issues) =================
      // runs up to VSTAGES stages ahead of the converter, independent of the MMAs
      uint32_t it = 0;
      for (int64_t w = blockIdx.x; w < n_items; w += gridDim.x) {
        const int blk = (int)(w % n_nblk);
        const int m0 = (int)(w / n_nblk) * BM;
        for (int q = 0; q < Q; ++q)
          for (int kc = 0; kc < KS; ++kc, ++it) {
            const uint32_t s = it % VSTAGES;
            if (it >= VSTAGES) PWAIT(0, &S.v_empty[s], ((it - VSTAGES) / VSTAGES) & 1);
            if (elect_one()) {
              const int na = stage_atoms(C, kc);
              if (PFLAG(8)) mbar_arrive(&S.v_full[s]);
              else {
                mbar_arrive_expect_tx(&S.v_full[s], na * V_ATOM_BYTES);
                for (int h = 0; h < na; ++h) tma_load_3d(S.v[s][h], &map_v, &S.v_full[s], SK * kc + VK * h, m0, q);
              }
              // V comes from HBM (the input transform just wrote it): prefetch
              // the V box of stage it + V_PREFETCH into L2.  pf_all == 0: once
              // per m-block -- the n_nblk CTAs of an m-block (running side by
              // side) take turns by stage, so L2 sees no redundant prefetch
              // requests; pf_all == 1 (many-frequency plans, where the CTAs of
              // an m-block drift further apart than L2 keeps V): every CTA
              if (V_PREFETCH > 0 && !PFLAG(8) && (pf_all || (int)((it + V_PREFETCH) % n_nblk) == blk)) {
                int nq = q, nk = kc + V_PREFETCH, nm = m0;
                nq += nk / KS;
                nk %= KS;
                if (nq >= Q) {
                  nq -= Q;
                  nm = (int)((w + gridDim.x) / n_nblk) * BM;
                }
                if (nm < d.tiles && nq < Q)
                  for (int h = 0; h < stage_atoms(C, nk); ++h) tma_prefetch_3d(&map_v, SK * nk + VK * h, nm, nq);
              }
            }
            __syncwarp();
          }
      }
    } else if (warp == WARP_UTMA) {
      // ================= U TMA producer: [U'hi; U'lo] of (frequency, 64 channels, n-block) =================
#if DWM_TC_U_EVICT_LAST
      const uint64_t upol = l2_policy_evict_last();
#endif
      uint32_t it = 0;
      for (int64_t w = blockIdx.x; w < n_items; w += gridDim.x) {
        const int blk = (int)(w % n_nblk);
        for (int q = 0; q < Q; ++q)
          for (int kc = 0; kc < KS; ++kc, ++it) {
            const uint32_t s = it % USTAGES;
            if (it >= USTAGES) mbar_wait(&S.done[(it - USTAGES) % STAGES], ((it - USTAGES) / STAGES) & 1);
            if (elect_one()) {
              // the U box is always full (channels past C are TMA zero fill)
              mbar_arrive_expect_tx(&S.u_full[s], U_ATOM_BYTES);
#if DWM_TC_U_EVICT_LAST
              // U is re-read by every m-block: keep it in L2 against the V stream
              tma_load_2d_hint(S.u[s], &map_u, &S.u_full[s], SK * kc, (q * n_nblk + blk) * (2 * BN), upol);
#else
              tma_load_2d(S.u[s], &map_u, &S.u_full[s], SK * kc, (q * n_nblk + blk) * (2 * BN));
#endif
            }
            __syncwarp();
          }
      }
    } else if (warp == WARP_MMA) {
      // ================= MMA issuer (whole warp converged, one lane issues) =================
      // one tcgen05.commit per 64-channel stage (each commit costs the tensor
      // pipe a ~140-cycle bubble, tools/commit_probe.cu)
      const uint32_t idesc128 = idesc_f16(BM, 2 * BN), idesc64 = idesc_f16(BM, BN);
      uint32_t it = 0, chunk = 0;
      for (int64_t w = blockIdx.x; w < n_items; w += gridDim.x) {
        for (int q = 0; q < Q; ++q) {
          for (int kc = 0; kc < KS; ++kc, ++it) {
            const uint32_t sb = it % STAGES, su = it % USTAGES, sa = it % A_SLOTS;
            const int na = stage_atoms(C, kc);
            const bool first = kc % CHS == 0;  // a chunk starts: fresh accumulators in buffer chunk % 2
            const uint32_t buf = chunk & 1u;
            if (first) PWAIT(0, &S.acc_empty[buf], ((chunk >> 1) & 1) ^ 1);
            PWAIT(1, &S.a_full[sa], (it / A_SLOTS) & 1);
            PWAIT(2, &S.u_full[su], (it / USTAGES) & 1);
            tc_fence_after();
            const uint32_t a_hi = tmem + COL_A + sa * A_COLS, a_lo = a_hi + A_COLS / 2;
            const uint32_t dacc = tmem + COL_ACC + buf * (2 * BN);
            if (elect_one()) {
              const uint64_t du = sdesc_sw128(smem_u32(S.u[su]));
              for (int k = 0; k < 2 * na; ++k) {
                // +32 B per K = 16 slice, in 16-byte descriptor units
                mma_f16_ts(dacc, a_hi + 8 * k, du + 2 * k, idesc128, (first && k == 0) ? 0u : 1u);
                if (!PFLAG(4)) mma_f16_ts(dacc + BN, a_lo + 8 * k, du + 2 * k, idesc64, 1u);
              }
              mma_commit(&S.done[sb]);
            }
            __syncwarp();
            if (kc % CHS == CHS - 1 || kc == KS - 1) ++chunk;
          }
        }
      }
    }
  } else if (warp < CONV_WARPS) {
    setmaxnreg_dec<REG_CONV>();
    // ================= converter: V stage (smem) -> s_v V -> hi/lo fp16 -> TMEM A slot =================
    // TMEM lane quadrant warp % 4 (rows m); with 8 warps, V atom warp / 4 (32 channels) each
    const uint32_t lane_addr = tmem + ((uint32_t)(32 * (warp % 4)) << 16);
    const int m = 32 * (warp % 4) + lane;
    const int h0 = CONV_WARPS == 8 ? warp / 4 : 0, hstep = CONV_WARPS == 8 ? 2 : 1;
    uint32_t it = 0;
    for (int64_t w = blockIdx.x; w < n_items; w += gridDim.x) {
      const float sv = exp2i(row_scale_exp(w, m));
      const f2 sv2 = pk(sv, sv);
      for (int q = 0; q < Q; ++q) {
        for (int kc = 0; kc < KS; ++kc, ++it) {
          const uint32_t sb = it % VSTAGES, sa = it % A_SLOTS;
          const int na = stage_atoms(C, kc);
          PWAIT(0, &S.v_full[sb], (it / VSTAGES) & 1);
          // A slot sa was last read by the MMAs of stage it - A_SLOTS
          if (it >= A_SLOTS) PWAIT(1, &S.done[(it - A_SLOTS) % STAGES], ((it - A_SLOTS) / STAGES) & 1);
          tc_fence_after();
          const uint32_t base = lane_addr + COL_A + sa * A_COLS;
          for (int h = h0; h < na; h += hstep) {
            if (PFLAG(1)) break;
            const uint32_t vrow = smem_u32(S.v[sb][h]);
            // the atom's 32 channels of row m: all 8 loads first (the loads are
            // volatile asm, so they would otherwise wait behind the previous
            // group's tcgen05.st), then the split, then two 16-column stores
            f2 xv[16];
#pragma unroll
            for (int c8 = 0; c8 < 8; ++c8)
              asm volatile("ld.shared.v2.b64 {%0, %1}, [%2];"
                           : "=l"(xv[2 * c8]), "=l"(xv[2 * c8 + 1])
                           : "r"(vrow + sw128_offset(m, 4 * c8)));
            uint32_t hi[16], lo[16];
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              // a channel pair, scaled, split and packed with f32x2 / f16x2 ops
              const float2 p = upk(mul2(xv[e], sv2));
              const __half2 h2 = __float22half2_rn(p);
              const uint32_t hu = *reinterpret_cast<const uint32_t*>(&h2);
              const __half2 l2 = __float22half2_rn(residual_f16x2(hu, p));
              hi[e] = hu;
              lo[e] = *reinterpret_cast<const uint32_t*>(&l2);
            }
            // channels 32 h + [0, 32) -> columns 16 h + [0, 16)
            tmem_st16u(base + 16 * h, hi);
            tmem_st16u(base + A_COLS / 2 + 16 * h, lo);
          }
          // every V value of the stage is in registers (consumed above): free the V slot
          __syncwarp();
          if (lane == 0) mbar_arrive(&S.v_empty[sb]);
          tmem_st_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&S.a_full[sa]);
        }
      }
    }
  } else {
    setmaxnreg_inc<REG_EPI>();
    // ================= epilogue: chunks -> M'_q -> Y (registers) -> y =================
    const int quad = warp % 4;
    const int c0 = ((warp - EPI_WARP0) / 4) * EC;
    const uint32_t lane_addr = tmem + ((uint32_t)(32 * quad) << 16);
    const int m = 32 * quad + lane;
    uint32_t it = 0, chunk = 0;
    for (int64_t w = blockIdx.x; w < n_items; w += gridDim.x) {
      const float inv_v = exp2i(-row_scale_exp(w, m));
      const int64_t tile = (w / n_nblk) * BM + m;
      const int n0 = (int)(w % n_nblk) * BN;
      float Y[4][EC];
#pragma unroll
      for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int j = 0; j < EC; ++j) Y[p][j] = 0.f;
      for (int q = 0; q < Q; ++q) {
        // output transform below: Y_p +-= M'_q for the positions p with a
        // nonzero coefficient (2-bit codes: 1 -> +1, 3 -> -1)
        const uint32_t cf = S.coef[q];
        float mq[EC];
        for (int kc = 0; kc < KS; ++kc, ++it) {
          if (!(kc % CHS == CHS - 1 || kc == KS - 1)) continue;  // chunk not complete yet
          PWAIT(0, &S.done[it % STAGES], (it / STAGES) & 1);
          tc_fence_after();
          const uint32_t buf = chunk & 1u;
          const bool first = kc < CHS;
          const uint32_t acc = lane_addr + COL_ACC + buf * (2 * BN) + c0;
#pragma unroll
          for (int h = 0; h < EC / 8; ++h) {
            if (PFLAG(2)) continue;
            float mn[8], cr[8];
            tmem_ld8(acc + 8 * h, mn);
            tmem_ld8(acc + BN + 8 * h, cr);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const float part = __fadd_rn(CHS == 1 ? trunc_compensate(mn[j], 1u) : mn[j], cr[j]);
              mq[8 * h + j] = first ? part : __fadd_rn(mq[8 * h + j], part);
            }
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&S.acc_empty[buf]);
          ++chunk;
        }
#pragma unroll
        for (int p = 0; p < 4; ++p) {
          const uint32_t code = (cf >> (2 * p)) & 3u;
          if (code == 1u) {
#pragma unroll
            for (int j = 0; j < EC; ++j) Y[p][j] = __fadd_rn(Y[p][j], mq[j]);
          } else if (code == 3u) {
#pragma unroll
            for (int j = 0; j < EC; ++j) Y[p][j] = __fsub_rn(Y[p][j], mq[j]);
          }
        }
      }
      // Y -> y: positions (i, j) of tile (n, ty, tx), this warp's filters, unscaled
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
          const float inv = __ldg(inv_f + f);
          float* yf = y + ((size_t)n * F + f) * (size_t)d.oh * d.ow + (size_t)oy * d.ow + ox;
#pragma unroll
          for (int ii = 0; ii < 2; ++ii) {
            if (oy + ii >= d.oh) continue;
            const float v0 = (Y[2 * ii][j] * inv_v) * inv, v1 = (Y[2 * ii + 1][j] * inv_v) * inv;
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
    const int role = warp == WARP_TMA ? 0 : warp == WARP_MMA ? 1 : warp == 0 ? 2 : warp == EPI_WARP0 ? 3 : -1;
    if (role >= 0 && lane == 0) {
      atomicAdd(&g_tc_prof[role * 4 + 0], (unsigned long long)prof[0]);
      atomicAdd(&g_tc_prof[role * 4 + 1], (unsigned long long)prof[1]);
      atomicAdd(&g_tc_prof[role * 4 + 2], (unsigned long long)prof[2]);
      atomicAdd(&g_tc_prof[role * 4 + 3], (unsigned long long)(clock64() - t_start));
    }
  }
#endif
  tc_fence_before();
  __syncthreads();
  if (warp == WARP_MMA) tmem_dealloc<512>(tmem);
}

// Per-image max|V| into the slots (the stage API's dwm_gemm_output gets V
// without the input transform's max|x|; |V| itself is a valid bound for the
// scale): one warp per (frequency, tile) row of C values.
__global__ void v_absmax_kernel(const dwm_desc_t d, const float* __restrict__ V, uint32_t* __restrict__ slots) {
  const int64_t rows = (int64_t)d.num_freqs * d.tiles, tiles_img = (int64_t)d.th * d.tw;
  const int lane = threadIdx.x % 32;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32; r < rows;
       r += (int64_t)gridDim.x * blockDim.x / 32) {
    uint32_t m = 0;
    for (int c = lane; c < d.c; c += 32) m = max(m, __float_as_uint(fabsf(V[r * d.c + c])));
    m = __reduce_max_sync(0xffffffffu, m);
    if (lane == 0) atomicMax(slots + (r % d.tiles) / tiles_img, m);
  }
}

// Per-filter scale s_f = 2^(12 - floor(log2 max|w_f|)) (stored as 1 / s_f),
// one CTA per (padded) filter; rows past F get 1.
__global__ void filter_scale_kernel(const dwm_desc_t d, const float* __restrict__ w, FiltView fv,
                                    float* __restrict__ inv_f) {
  const int f = blockIdx.x;
  uint32_t m = 0;
  if (f < d.f) {
    const int taps = d.r_h * d.r_w, n = d.c * taps;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const int c = i / taps, t = i % taps;
      const float v = w[(int64_t)f * fv.sf + (int64_t)c * fv.sc + (int64_t)(t / d.r_w) * fv.skh + (int64_t)(t % d.r_w) * fv.skw];
      m = max(m, __float_as_uint(fabsf(v)));
    }
  }
  m = __reduce_max_sync(0xffffffffu, m);
  __shared__ uint32_t red[32];
  if (threadIdx.x % 32 == 0) red[threadIdx.x / 32] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < (int)blockDim.x / 32; ++i) m = max(m, red[i]);
    m = max(m, red[0]);
    inv_f[f] = exp2i(-scale_exp(m));
  }
}

// U'hi / U'lo (fp16) per 64-filter block, stacked:
// U[((fq * nblk + f / 64) * 128 + {0: hi, 64: lo} + f % 64) * C + c]; one
// thread per (f, c) over the padded filter count (rows past F are zeros).
__global__ void filter_split_kernel(const dwm_desc_t d, const float* __restrict__ w, FiltView fv,
                                    const float* __restrict__ inv_f, __half* __restrict__ U) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int nblk = (d.f + BN - 1) / BN;
  const int64_t fcp = (int64_t)nblk * BN * d.c;
  if (idx >= fcp) return;
  const int f = (int)(idx / d.c), c = (int)(idx % d.c);
  const bool live = f < d.f;
  const float s = __frcp_rn(inv_f[f]);
  const int64_t row0 = (int64_t)(f / BN) * (2 * BN) + f % BN;
  int fq = 0;
  for (int rp = 0; rp < d.n_row_parts; ++rp)
    for (int cp = 0; cp < d.n_col_parts; ++cp) {
      float u[4][4];
      part_filter_transform(d, w + (live ? (int64_t)f * fv.sf + (int64_t)c * fv.sc : 0), fv, rp, cp, u);
      const int lr = d.row_parts[rp].count + 1, lc = d.col_parts[cp].count + 1;
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b)
          if (a < lr && b < lc) {
            const float v = live ? u[a][b] * s : 0.f;
            const __half hi = __float2half_rn(v);
            const __half lo = __float2half_rn(v - __half2float(hi));
            const int64_t o = ((int64_t)(fq + a * lc + b) * nblk * (2 * BN) + row0) * d.c + c;
            U[o] = hi;
            U[o + (int64_t)BN * d.c] = lo;
          }
      fq += lr * lc;
    }
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
  const cuuint32_t box[3] = {VK, BM, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, (void*)base, dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(DWM_ECUDA, "cuTensorMapEncodeTiled(V) failed (%d)", (int)r);
  return DWM_OK;
}

// U in the stacked layout: [freq][64-filter block][U'hi 64 rows; U'lo 64 rows][C] fp16
int make_u_map(CUtensorMap* map, const void* base, const dwm_desc_t& d) {
  auto encode = get_encode();
  if (!encode) return fail(DWM_ECUDA, "cuTensorMapEncodeTiled is unavailable");
  const int64_t nblk = (d.f + BN - 1) / BN;
  const cuuint64_t dims[2] = {(cuuint64_t)d.c, (cuuint64_t)(d.num_freqs * nblk * 2 * BN)};
  const cuuint64_t strides[1] = {(cuuint64_t)d.c * 2};
  const cuuint32_t box[2] = {SK, 2 * BN};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, (void*)base, dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(DWM_ECUDA, "cuTensorMapEncodeTiled(U) failed (%d)", (int)r);
  return DWM_OK;
}

size_t u_split_bytes(const dwm_desc_t& d) {
  return (size_t)d.num_freqs * (size_t)((d.f + BN - 1) / BN) * 2 * BN * (size_t)d.c * 2;
}

}  // namespace

bool tc_gemm_supported(const dwm_desc_t& d) {
  return d.c % VK == 0 && d.f >= 1 && d.num_freqs <= MAX_FREQS && d.tiles < ((int64_t)1 << 31);
}

// [U'hi; U'lo] fp16 planes, then one fp32 1 / s_f per padded filter
size_t tc_filter_bytes(const dwm_desc_t& d) {
  return u_split_bytes(d) + (size_t)((d.f + BN - 1) / BN) * BN * sizeof(float);
}

int launch_filter_transform_f16split(const dwm_desc_t& d, const void* w, void* U, cudaStream_t s,
                                     const int64_t* strides) {
  const FiltView fv = strides ? FiltView{strides[0], strides[1], strides[2], strides[3]}
                                 : FiltView{(int64_t)d.c * d.r_h * d.r_w, (int64_t)d.r_h * d.r_w, d.r_w, 1};
  const int nblk = (d.f + BN - 1) / BN;
  float* inv_f = reinterpret_cast<float*>(static_cast<char*>(U) + u_split_bytes(d));
  filter_scale_kernel<<<nblk * BN, 256, 0, s>>>(d, (const float*)w, fv, inv_f);
  const int64_t n = (int64_t)nblk * BN * d.c;
  filter_split_kernel<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(d, (const float*)w, fv, inv_f, (__half*)U);
  DWM_CUDA_TRY(cudaGetLastError());
  return DWM_OK;
}

// Accumulator chunk: 128 channels (2 stages) when C >= 128, else 64 channels
// with the +1 ulp compensation.  DWM_TC_CHUNK=64|128 overrides (experiments).
static int tc_chunk_stages(const dwm_desc_t& d) {
  static const int env = [] {
    const char* e = getenv("DWM_TC_CHUNK");
    return e ? atoi(e) : 0;
  }();
  if (env == 64) return 1;
  if (env == 128) return 2;
  return d.c >= 128 ? 2 : 1;
}

int launch_gemm_tc(const dwm_desc_t& d, const void* V, const void* U, void* y, int32_t* flag, const uint32_t* xmax,
                   void* scratch, size_t scratch_bytes, cudaStream_t s) {
  if (!tc_gemm_supported(d)) return fail(DWM_EUNSUPPORTED, "tcgen05 GEMM needs C %% 32 == 0");
  if (!xmax) {
    // no input-transform range: bound the scale by max|V| itself
    if (!scratch || scratch_bytes < xmax_bytes(d))
      return fail(DWM_EINVAL_SHAPE, "tcgen05 GEMM on a caller V needs %zu bytes of workspace (4 per image, got %zu)",
                  xmax_bytes(d), scratch_bytes);
    DWM_CUDA_TRY(cudaMemsetAsync(scratch, 0, xmax_bytes(d), s));
    v_absmax_kernel<<<1184, 256, 0, s>>>(d, (const float*)V, (uint32_t*)scratch);
    xmax = (const uint32_t*)scratch;
  }
  CUtensorMap mv, mu;
  if (int st = make_v_map(&mv, (const float*)V, d)) return st;
  if (int st = make_u_map(&mu, U, d)) return st;
  const float* inv_f = reinterpret_cast<const float*>(static_cast<const char*>(U) + u_split_bytes(d));
  const size_t smem = sizeof(Smem) + 1024;
  int sms = 0;
  if (int st = device_sm_count(&sms)) return st;
  const int64_t items = ((d.tiles + BM - 1) / BM) * ((d.f + BN - 1) / BN);
  const int grid = (int)(items < sms ? items : sms);
  // V prefetch by every CTA above this many frequencies: cfg4 11x11 (225
  // frequencies) GEMM DRAM reads 52 -> 25 GB and 15.25 -> 14.86 ms at higher
  // clocks (less DRAM power); turns win below: cfg4 9x9 (144) 8.9-9.2 vs
  // 9.4-9.6 ms, 7x7 (100) 5.67 vs 6.15-6.22 ms (profiles/r2/ab_tc_prefetch_all.txt).
  // DWM_TC_PF_ALL_Q overrides the threshold.
  static const int pf_q = [] {
    const char* e = getenv("DWM_TC_PF_ALL_Q");
    return e ? atoi(e) : 200;
  }();
  const int pf_all = d.num_freqs > pf_q ? 1 : 0;
  if (tc_chunk_stages(d) == 2) {
    if (int st = ensure_dynamic_smem((const void*)gemm_tc_kernel<2>, smem)) return st;
    gemm_tc_kernel<2><<<grid, THREADS, smem, s>>>(d, mv, mu, inv_f, xmax, (float*)y, flag, pf_all);
  } else {
    if (int st = ensure_dynamic_smem((const void*)gemm_tc_kernel<1>, smem)) return st;
    gemm_tc_kernel<1><<<grid, THREADS, smem, s>>>(d, mv, mu, inv_f, xmax, (float*)y, flag, pf_all);
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
