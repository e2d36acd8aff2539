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
// hi = rn_tf32(x), lo = rn_tf32(x - hi) (the tensor core would truncate a raw
// fp32 operand; tools/tc_probe.cu measured that).  U_hi/U_lo come pre-split
// from the filter transform; V is split on the fly.
//
// Accumulation accuracy: the tcgen05 FP32 accumulator rounds toward zero
// (tools/tc_accum_probe.cu: -0.54 ulp per MMA step, biased), so a long MMA
// chain into one accumulator is ~25x worse in MSE than the reference's RN FMA
// chain.  Each 32-channel chunk therefore gets a fresh TMEM accumulator: its 8
// small correction MMAs (hi*lo, lo*hi) go first, while the accumulator is
// still small, then its main MMAs (hi*hi); the epilogue sums the chunks in
// FP32 round-to-nearest.  Emulated MSE vs the reference: 0.2-0.4x.  (Chunks
// are 16 channels, the granularity of the 4-deep TMEM A-operand ring.)
//   Y_(i,j) += At_r[i][a] * At_c[j][b] * M_q     (coefficients 0, +-1)
// and only y = interleave(Y) reaches HBM.
//
// Warp roles (448 threads, one CTA per SM, persistent over work items):
//   warps 0-3  converter: V row (one tile per thread) from the smem stage ->
//              hi/lo -> tcgen05.st into a TMEM A-operand stage (double buffered)
//   warps 4-11 epilogue : tcgen05.ld each chunk -> M_q (registers, FP32 RN);
//              +-add M_q into the TMEM Y accumulators; at the end of a work
//              item Y -> y (NCHW), non-finite flag.  Two warps per TMEM lane
//              quadrant, 32 filter columns each.
//   warp 12    TMA producer: V tile [128 tiles][32 ch] and U_hi/U_lo tiles
//              [64 f][32 ch] per (frequency, chunk) stage (SWIZZLE_128B, 6 stages)
//   warp 13    TMEM allocator + tcgen05.mma issuer (TS mode: A = V from TMEM,
//              B = U from smem), commits to mbarriers; issue from the
//              converged warp via elect.sync
// TMEM columns: chunk acc[2] 0-127, A stages 128-255 (4 x [hi 16 | lo 16]), Y 256-511.
#include <cuda.h>
#include <unistd.h>
#include <cstdio>
#include <cudaTypedefs.h>

#include "dwm_common.cuh"
#include "dwm_kernels.h"
#include "dwm_sm100.cuh"

namespace dwm {
namespace {

using namespace sm100;

constexpr int BM = 128;        // tiles per work item (MMA M, TMEM lanes)
constexpr int BN = 64;         // filters per work item (MMA N)
constexpr int BK = 32;         // channels per stage (128 B rows, one SW128 atom)
constexpr int B_STAGES = 6;
#ifndef DWM_TC_AK
#define DWM_TC_AK 32
#endif
constexpr int AK = DWM_TC_AK;       // channels per A stage / per accumulator chunk
constexpr int A_STAGES = 64 / AK;   // TMEM A-operand ring in 128 columns (hi AK | lo AK each)
constexpr int THREADS = 448;    // 4 converter + 8 epilogue + TMA + MMA warps
constexpr int EPI_WARPS = 8;
constexpr int EC = BN / (EPI_WARPS / 4);  // columns per epilogue warp (32)
constexpr int WARP_TMA = 12, WARP_MMA = 13;
constexpr int MAX_FREQS = 1024;
constexpr uint32_t U_TILE_BYTES = BN * BK * 4;  // 8 KB per plane
constexpr uint32_t V_TILE_BYTES = BM * BK * 4;  // 16 KB
constexpr uint32_t COL_ACC = 0, COL_A = 128, COL_Y = 256;

// Debug builds (-DDWM_TC_TRACE) publish per-role progress into mapped host
// memory so a stuck pipeline can be diagnosed while the kernel still runs.
#ifdef DWM_TC_TRACE
#define TRACE(slot, val) do { if (trace) { trace[slot] = (val); __threadfence_system(); } } while (0)
// per-role cycles spent blocked in mbarrier waits (block 0, one thread per role)
#define TWAIT(acc, bar, ph) do { long long _t0 = clock64(); mbar_wait(bar, ph); acc += clock64() - _t0; } while (0)
#else
#define TRACE(slot, val) do { } while (0)
#define TWAIT(acc, bar, ph) mbar_wait(bar, ph)
#endif

struct __align__(1024) Smem {
  float v[B_STAGES][BM * BK];
  float u_hi[B_STAGES][BN * BK];
  float u_lo[B_STAGES][BN * BK];
  uint64_t b_full[B_STAGES], b_empty[B_STAGES];
  uint64_t a_full[A_STAGES], a_empty[A_STAGES];
  uint64_t acc_full[2], acc_empty[2];
  uint32_t tmem_base;
  int8_t coef[MAX_FREQS][4];
};

__device__ __forceinline__ int at_coef_rt(int r, int i, int a) {
  return r == 1 ? (i == a ? 1 : 0)
       : r == 2 ? (i == 0 ? (a <= 1 ? 1 : 0) : (a == 1 ? 1 : (a == 2 ? -1 : 0)))
                : (i == 0 ? (a <= 2 ? 1 : 0) : (a == 0 ? 0 : (a == 1 ? 1 : -1)));
}

__global__ void __launch_bounds__(THREADS, 1)
gemm_tc_kernel(const dwm_desc_t d, const __grid_constant__ CUtensorMap map_v, const __grid_constant__ CUtensorMap map_uhi,
               const __grid_constant__ CUtensorMap map_ulo, float* __restrict__ y, int32_t* __restrict__ flag,
               volatile int* trace) {
  extern __shared__ uint8_t smem_raw[];
  Smem& S = *reinterpret_cast<Smem*>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const int Q = d.num_freqs, C = d.c, F = d.f;
  const int KC = C / BK;
  const int n_nblk = (F + BN - 1) / BN;  // a partial last block computes garbage columns, never stored
  const int64_t n_mblk = (d.tiles + BM - 1) / BM;
  const int64_t n_items = n_mblk * n_nblk;

  // ---- one-time setup
  if (tid == 0) {
    for (int i = 0; i < B_STAGES; ++i) {
      mbar_init(&S.b_full[i], 1);
      mbar_init(&S.b_empty[i], 1 + 4);  // MMA commit (U) + 4 converter warps (V)
    }
    for (int i = 0; i < A_STAGES; ++i) {
      mbar_init(&S.a_full[i], 4);
      mbar_init(&S.a_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&S.acc_full[i], 1);
      mbar_init(&S.acc_empty[i], EPI_WARPS);
    }
    fence_barrier_init();
    // output-transform coefficient of every frequency for the 4 tile positions
    int q = 0;
    for (int rp = 0; rp < d.n_row_parts; ++rp)
      for (int cp = 0; cp < d.n_col_parts; ++cp) {
        const int pr = d.row_parts[rp].count, pc = d.col_parts[cp].count;
        for (int a = 0; a <= pr; ++a)
          for (int b = 0; b <= pc; ++b, ++q)
            for (int i = 0; i < 2; ++i)
              for (int j = 0; j < 2; ++j) S.coef[q][i * 2 + j] = (int8_t)(at_coef_rt(pr, i, a) * at_coef_rt(pc, j, b));
      }
  }
  if (warp == WARP_TMA && lane == 0) {
    tma_prefetch_desc(&map_v);
    tma_prefetch_desc(&map_uhi);
    tma_prefetch_desc(&map_ulo);
  }
  if (warp == WARP_MMA) tmem_alloc<512>(&S.tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = S.tmem_base;
  if (tid == 0 && blockIdx.x == 0) TRACE(0, 1);
#ifdef DWM_TC_TRACE
  long long w_tma = 0, w_mma_b = 0, w_mma_acc = 0, w_mma_a = 0, w_cv_b = 0, w_cv_a = 0, w_ep = 0;
  const long long t_start = clock64();
#endif

  if (warp == WARP_TMA) {
    // ================= TMA producer (whole warp converged, one lane issues) =================
    uint32_t it = 0;
    for (int64_t w = blockIdx.x; w < n_items; w += gridDim.x) {
      const int n0 = (int)(w % n_nblk) * BN;
      const int m0 = (int)(w / n_nblk) * BM;
      for (int q = 0; q < Q; ++q)
        for (int kc = 0; kc < KC; ++kc, ++it) {
          const uint32_t s = it % B_STAGES, round = it / B_STAGES;
          TWAIT(w_tma, &S.b_empty[s], (round & 1) ^ 1);
          if (elect_one()) {
#if defined(DWM_EXP_NO_V_LOAD)
            mbar_arrive_expect_tx(&S.b_full[s], 2 * U_TILE_BYTES);
            tma_load_2d(S.u_hi[s], &map_uhi, &S.b_full[s], kc * BK, q * F + n0);
            tma_load_2d(S.u_lo[s], &map_ulo, &S.b_full[s], kc * BK, q * F + n0);
#elif defined(DWM_EXP_NO_U_LOAD)
            mbar_arrive_expect_tx(&S.b_full[s], V_TILE_BYTES);
            tma_load_3d(S.v[s], &map_v, &S.b_full[s], kc * BK, m0, q);
#else
            mbar_arrive_expect_tx(&S.b_full[s], V_TILE_BYTES + 2 * U_TILE_BYTES);
            tma_load_3d(S.v[s], &map_v, &S.b_full[s], kc * BK, m0, q);
            tma_load_2d(S.u_hi[s], &map_uhi, &S.b_full[s], kc * BK, q * F + n0);
            tma_load_2d(S.u_lo[s], &map_ulo, &S.b_full[s], kc * BK, q * F + n0);
#endif
          }
          __syncwarp();
        }
    }
  } else if (warp == WARP_MMA) {
    // ================= MMA issuer (whole warp converged, one lane issues) =================
    {
      const uint32_t idesc = idesc_tf32(BM, BN);
      uint32_t itb = 0, ita = 0;
      for (int64_t w = blockIdx.x; w < n_items; w += gridDim.x) {
        for (int q = 0; q < Q; ++q) {
          for (int kc = 0; kc < KC; ++kc, ++itb) {
            const uint32_t sb = itb % B_STAGES;
            // no b_full wait: the converter only signals a_full after it
            // observed b_full, and the same TMA transaction carried the U tiles
            const uint64_t dh0 = sdesc_sw128(smem_u32(S.u_hi[sb])), dl0 = sdesc_sw128(smem_u32(S.u_lo[sb]));
#pragma unroll
            for (int h = 0; h < BK / AK; ++h, ++ita) {
              // one fresh accumulator per AK-channel chunk (ring of 2)
              const uint32_t ab = ita % 2, sa = ita % A_STAGES;
              const uint32_t dacc = tmem + COL_ACC + ab * BN;
              TWAIT(w_mma_acc, &S.acc_empty[ab], ((ita / 2) & 1) ^ 1);
              TWAIT(w_mma_a, &S.a_full[sa], (ita / A_STAGES) & 1);
              tc_fence_after();
              const uint32_t a_hi = tmem + COL_A + sa * (2 * AK), a_lo = a_hi + AK;
              if (elect_one()) {
                // small correction products first, while the accumulator is small
#pragma unroll
                for (int k = 0; k < AK / 8; ++k) {
                  const uint32_t kd = 2 * (h * (AK / 8) + k);  // +32 B per K=8 slice, in 16-byte descriptor units
                  mma_tf32_ts(dacc, a_hi + 8 * k, dl0 + kd, idesc, k != 0);
                  mma_tf32_ts(dacc, a_lo + 8 * k, dh0 + kd, idesc, 1);
                }
#pragma unroll
                for (int k = 0; k < AK / 8; ++k) mma_tf32_ts(dacc, a_hi + 8 * k, dh0 + 2 * (h * (AK / 8) + k), idesc, 1);
                mma_commit(&S.a_empty[sa]);
                mma_commit(&S.acc_full[ab]);
              }
              __syncwarp();
            }
            if (elect_one()) mma_commit(&S.b_empty[sb]);
            __syncwarp();
          }
        }
      }
    }
  } else if (warp < 4) {
    // ================= converter: V stage (smem) -> hi/lo -> TMEM A stage =================
    const uint32_t lane_addr = tmem + ((uint32_t)(32 * warp) << 16);
    const int m = 32 * warp + lane;
    uint32_t ita = 0, ita2 = 0;
    for (int64_t w = blockIdx.x; w < n_items; w += gridDim.x) {
      for (int q = 0; q < Q; ++q) {
        for (int kc = 0; kc < KC; ++kc, ++ita) {
          const uint32_t sb = ita % B_STAGES;
          TWAIT(w_cv_b, &S.b_full[sb], (ita / B_STAGES) & 1);
          float hi[32], lo[32];
          const uint8_t* vrow = reinterpret_cast<const uint8_t*>(S.v[sb]);
#pragma unroll
          for (int c4 = 0; c4 < 8; ++c4) {
            // row m, 16-byte chunk c4 of the SWIZZLE_128B tile
            const float4 x = *reinterpret_cast<const float4*>(vrow + sw128_offset(m, 4 * c4));
            const float xs[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              // hi = tf32 round-to-nearest (ties away) in 2 integer ops; lo = x - hi
              // exactly, handed to the tensor core raw (it truncates lo to tf32:
              // emulated MSE identical to an RN lo, tools/../DESIGN.md §3.1)
              const float h = __uint_as_float((__float_as_uint(xs[e]) + 0x1000u) & 0xFFFFE000u);
              hi[c4 * 4 + e] = h;
              lo[c4 * 4 + e] = __fsub_rn(xs[e], h);
            }
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&S.b_empty[sb]);  // this warp is done with the V rows
#pragma unroll
          for (int h = 0; h < BK / AK; ++h) {
            const uint32_t sa = ita2 % A_STAGES;
            TWAIT(w_cv_a, &S.a_empty[sa], ((ita2 / A_STAGES) & 1) ^ 1);
            tc_fence_after();
            const uint32_t base = lane_addr + COL_A + sa * (2 * AK);
#ifndef DWM_EXP_NO_CONV_ST
            static_assert(AK == 32, "one x32 TMEM store per operand half");
            tmem_st32(base, *reinterpret_cast<float(*)[32]>(hi + h * AK));
            tmem_st32(base + AK, *reinterpret_cast<float(*)[32]>(lo + h * AK));
#else
            if (hi[0] == 12345.f) tmem_st16(base, *reinterpret_cast<float(*)[16]>(hi));
#endif
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&S.a_full[sa]);
            ++ita2;
          }
        }
      }
    }
  } else {
    // ================= epilogue: M_q -> Y (TMEM) -> y =================
    // 8 warps: TMEM lane quadrant = warp % 4 (hardware rule), column half = (warp - 4) / 4
    const int quad = warp % 4;
    const int c0 = ((warp - 4) / 4) * EC;
    const uint32_t lane_addr = tmem + ((uint32_t)(32 * quad) << 16);
    const int m = 32 * quad + lane;
    uint32_t itq = 0;
    for (int64_t w = blockIdx.x; w < n_items; w += gridDim.x) {
      const int64_t tile = (w / n_nblk) * BM + m;
      const int n0 = (int)(w % n_nblk) * BN;
      // zero this warp's Y accumulators
      {
        float z[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) z[j] = 0.f;
#pragma unroll
        for (int p = 0; p < 4; ++p)
#pragma unroll
          for (int c = 0; c < EC; c += 16) tmem_st16(lane_addr + COL_Y + p * BN + c0 + c, z);
        tmem_st_wait();
      }
      for (int q = 0; q < Q; ++q) {
        float mq[EC];
        for (int kc = 0; kc < KC * (BK / AK); ++kc, ++itq) {
          const uint32_t ab = itq % 2;
          TWAIT(w_ep, &S.acc_full[ab], (itq / 2) & 1);
          tc_fence_after();
          float part[EC];
          static_assert(EC == 32, "one x32 TMEM load per epilogue warp and chunk");
          tmem_ld32(lane_addr + COL_ACC + ab * BN + c0, part);
          tmem_ld_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&S.acc_empty[ab]);
          if (kc == 0) {
#pragma unroll
            for (int j = 0; j < EC; ++j) mq[j] = part[j];
          } else {
#pragma unroll
            for (int j = 0; j < EC; ++j) mq[j] = __fadd_rn(mq[j], part[j]);
          }
        }
        // output transform: Y_p +-= M_q for the positions p with a nonzero coefficient
        const int8_t cf[4] = {S.coef[q][0], S.coef[q][1], S.coef[q][2], S.coef[q][3]};
#pragma unroll
        for (int p = 0; p < 4; ++p) {
#ifdef DWM_EXP_NO_EPI_Y
          if (mq[0] != 12345.f) continue;
#endif
          if (cf[p] == 0) continue;
          float yv[EC];
          const uint32_t ya = lane_addr + COL_Y + p * BN + c0;
          tmem_ld32(ya, yv);
          tmem_ld_wait();
          if (cf[p] > 0) {
#pragma unroll
            for (int j = 0; j < EC; ++j) yv[j] = __fadd_rn(yv[j], mq[j]);
          } else {
#pragma unroll
            for (int j = 0; j < EC; ++j) yv[j] = __fsub_rn(yv[j], mq[j]);
          }
#pragma unroll
          tmem_st32(ya, yv);
        }
        tmem_st_wait();
      }
      // Y -> y: positions (i, j) of tile (n, ty, tx), this warp's filters.
      // tcgen05.ld is warp-collective: every lane loads, only live tiles store.
      {
        const bool live = tile < d.tiles;
        const int64_t tl = live ? tile : 0;
        const int tx = (int)(tl % d.tw);
        const int64_t t2 = tl / d.tw;
        const int ty = (int)(t2 % d.th);
        const int n = (int)(t2 / d.th);
        bool bad = false;
#pragma unroll 1
        for (int ch = 0; ch < EC; ch += 16) {
          float y00[16], y01[16], y10[16], y11[16];
          tmem_ld16(lane_addr + COL_Y + 0 * BN + c0 + ch, y00);
          tmem_ld16(lane_addr + COL_Y + 1 * BN + c0 + ch, y01);
          tmem_ld16(lane_addr + COL_Y + 2 * BN + c0 + ch, y10);
          tmem_ld16(lane_addr + COL_Y + 3 * BN + c0 + ch, y11);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 16 && live; ++j) {
            const int f = n0 + c0 + ch + j;
            if (f >= F) break;
            float* yf = y + ((size_t)n * F + f) * (size_t)d.oh * d.ow;
            const int oy = 2 * ty, ox = 2 * tx;
            const float v[2][2] = {{y00[j], y01[j]}, {y10[j], y11[j]}};
#pragma unroll
            for (int ii = 0; ii < 2; ++ii) {
              if (oy + ii >= d.oh) continue;
              float* dst = yf + (size_t)(oy + ii) * d.ow + ox;
              if (ox + 1 < d.ow) {
                bad |= !(isfinite(v[ii][0]) && isfinite(v[ii][1]));
                if ((d.ow & 1) == 0 && ((uintptr_t)y & 7) == 0) {
                  __stcs(reinterpret_cast<float2*>(dst), make_float2(v[ii][0], v[ii][1]));
                } else {
                  __stcs(dst, v[ii][0]);
                  __stcs(dst + 1, v[ii][1]);
                }
              } else {
                bad |= !isfinite(v[ii][0]);
                __stcs(dst, v[ii][0]);
              }
            }
          }
        }
        if (bad && flag) *flag = 1;
      }
    }
  }

  if (blockIdx.x == 0 && lane == 0) TRACE(8 + warp, 1);
#ifdef DWM_TC_TRACE
  if (blockIdx.x == 0) {
    const long long tot = clock64() - t_start;
    if (tid == 0) { TRACE(20, (int)(tot >> 10)); TRACE(21, (int)(w_cv_b >> 10)); TRACE(22, (int)(w_cv_a >> 10)); }
    if (tid == 128) TRACE(23, (int)(w_ep >> 10));
    if (tid == 32 * WARP_TMA) TRACE(24, (int)(w_tma >> 10));
    if (tid == 32 * WARP_MMA) { TRACE(25, (int)(w_mma_b >> 10)); TRACE(26, (int)(w_mma_acc >> 10)); TRACE(27, (int)(w_mma_a >> 10)); }
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

int make_u_map(CUtensorMap* map, const float* base, const dwm_desc_t& d) {
  auto encode = get_encode();
  if (!encode) return fail(DWM_ECUDA, "cuTensorMapEncodeTiled is unavailable");
  const cuuint64_t dims[2] = {(cuuint64_t)d.c, (cuuint64_t)d.num_freqs * d.f};
  const cuuint64_t strides[1] = {(cuuint64_t)d.c * sizeof(float)};
  const cuuint32_t box[2] = {BK, BN};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)base, dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(DWM_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return DWM_OK;
}

}  // namespace

bool tc_gemm_supported(const dwm_desc_t& d) {
  // any F: U rows past a frequency's F read the next frequency's filters (or
  // TMA zero fill) and those accumulator columns are never stored
  return d.c % BK == 0 && d.f >= 1 && d.num_freqs <= MAX_FREQS && d.tiles < ((int64_t)1 << 31);
}

int launch_gemm_tc(const dwm_desc_t& d, const void* V, const void* U, void* y, int32_t* flag, cudaStream_t s) {
  if (!tc_gemm_supported(d)) return fail(DWM_EUNSUPPORTED, "tcgen05 GEMM needs C %% 32 == 0");
  const float* uhi = (const float*)U;
  const float* ulo = uhi + (size_t)d.num_freqs * d.f * d.c;
  CUtensorMap mv, mh, ml;
  if (int st = make_v_map(&mv, (const float*)V, d)) return st;
  if (int st = make_u_map(&mh, uhi, d)) return st;
  if (int st = make_u_map(&ml, ulo, d)) return st;
  const size_t smem = sizeof(Smem) + 1024;
  DWM_CUDA_TRY(cudaFuncSetAttribute(gemm_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int dev = 0, sms = 0;
  DWM_CUDA_TRY(cudaGetDevice(&dev));
  DWM_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int64_t items = ((d.tiles + BM - 1) / BM) * ((d.f + BN - 1) / BN);
  const int grid = (int)(items < sms ? items : sms);
#ifdef DWM_TC_TRACE
  static int* trace_h = nullptr;
  int* trace_d = nullptr;
  if (!trace_h) DWM_CUDA_TRY(cudaHostAlloc((void**)&trace_h, 64 * sizeof(int), cudaHostAllocMapped));
  for (int i = 0; i < 64; ++i) trace_h[i] = -1;
  DWM_CUDA_TRY(cudaHostGetDevicePointer((void**)&trace_d, trace_h, 0));
  gemm_tc_kernel<<<grid, THREADS, smem, s>>>(d, mv, mh, ml, (float*)y, flag, trace_d);
  DWM_CUDA_TRY(cudaGetLastError());
  for (int i = 0; i < 50 && cudaStreamQuery(s) == cudaErrorNotReady; ++i) usleep(100000);
  fprintf(stderr, "[tc trace] done=%d setup=%d tma_it=%d mma_q=%d mma_kc=%d conv=%d epi=%d exits:", 
          cudaStreamQuery(s) == cudaSuccess, trace_h[0], trace_h[1], trace_h[2], trace_h[3], trace_h[4], trace_h[5]);
  for (int w = 0; w < 10; ++w) fprintf(stderr, " %d", trace_h[8 + w]);
  fprintf(stderr, "\n[tc trace] kcycles total %d | conv wait V %d wait A-slot %d | epi wait acc %d | tma wait slot %d | "
          "mma wait U %d wait acc-slot %d wait A %d\n", trace_h[20], trace_h[21], trace_h[22], trace_h[23], trace_h[24],
          trace_h[25], trace_h[26], trace_h[27]);
#else
  gemm_tc_kernel<<<grid, THREADS, smem, s>>>(d, mv, mh, ml, (float*)y, flag, nullptr);
  DWM_CUDA_TRY(cudaGetLastError());
#endif
  return DWM_OK;
}

}  // namespace dwm
