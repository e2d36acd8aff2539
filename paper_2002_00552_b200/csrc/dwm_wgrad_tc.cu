// dwm_wgrad_tc.cu -- weight gradient of the DWM forward on the tcgen05 tensor
// cores, in the Winograd domain like the reference (
// reference _winograd_grad_weight_impl engines.py:258-330, placement
// engines.py:389-392):
//
//   DM_q[f][t]  = (A dY A^T)_q          per 2x2 output tile t, per frequency q
//   V_q[t][c]   = (B^T d B)_q           the forward's input transform
//   dU_q[c][f]  = sum_t V_q[t][c] * DM_q[f][t]          <- tcgen05, K = tiles
//   dg[f][c]    = G^T dU G per part, placed at the part's taps
//
// The contraction runs like the forward GEMM (dwm_gemm_tc.cu), transposed:
// M = 128 channels (TMEM lanes), N = 64 filters, K = tiles in chunks of 32,
// 3xTF32 (V split on the fly by the converter warps, DM pre-split by the
// grad-out transform), a fresh TMEM accumulator per 32-tile chunk (the TMEM
// accumulator truncates; see dwm_gemm_tc.cu), chunks summed in FP32
// round-to-nearest in a blocked order (64 chunks -> block sum -> total), so
// the K = N*TH*TW-long reduction never runs as one long chain.
//
// Warp roles (448 threads, persistent over (frequency, 128-channel block,
// 64-filter block) work items):
//   warps 0-3  converter: column `lane` of its 32x32 V box (channel c = 32w +
//              lane, tiles t = 0..31) -> hi/lo -> tcgen05.st (TMEM lane = c)
//   warps 4-11 epilogue : chunk accumulator -> blocked FP32 sums -> dU
//   warp 12    TMA producer: 4 V boxes [32 t][32 c] + DM_hi/DM_lo [64 f][32 t]
//   warp 13    TMEM allocator + MMA issuer (TS: A = V from TMEM, B = DM smem)
#include <cuda.h>
#include <cudaTypedefs.h>

#include "dwm_common.cuh"
#include "dwm_kernels.h"
#include "dwm_sm100.cuh"

namespace dwm {
namespace {

using namespace sm100;

constexpr int BM = 128;  // channels per work item (MMA M, TMEM lanes)
constexpr int BN = 64;   // filters per work item (MMA N)
constexpr int BK = 32;   // tiles per stage / per accumulator chunk
constexpr int B_STAGES = 6;
constexpr int A_STAGES = 2;
constexpr int THREADS = 448;
constexpr int EPI_WARPS = 8;
constexpr int EC = 32;
constexpr int WARP_TMA = 12, WARP_MMA = 13;
constexpr uint32_t VBOX_BYTES = 32 * 32 * 4;  // 4 KB, one per converter warp
constexpr uint32_t D_TILE_BYTES = BN * BK * 4;  // 8 KB per plane
constexpr uint32_t COL_ACC = 0, COL_A = 128;
constexpr int BLOCK_CHUNKS = 64;  // chunks per blocked partial sum

struct __align__(1024) WSmem {
  float v[B_STAGES][4][32 * 32];
  float d_hi[B_STAGES][BN * BK];
  float d_lo[B_STAGES][BN * BK];
  uint64_t b_full[B_STAGES], b_empty[B_STAGES];
  uint64_t a_full[A_STAGES], a_empty[A_STAGES];
  uint64_t acc_full[2], acc_empty[2];
  uint32_t tmem_base;
};

__global__ void __launch_bounds__(THREADS, 1)
wgrad_tc_kernel(const dwm_desc_t d, int64_t t_pad, const __grid_constant__ CUtensorMap map_v,
                const __grid_constant__ CUtensorMap map_dhi, const __grid_constant__ CUtensorMap map_dlo,
                float* __restrict__ du) {
  extern __shared__ uint8_t smem_raw[];
  WSmem& S = *reinterpret_cast<WSmem*>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const int C = d.c, F = d.f;
  const int n_cb = (C + BM - 1) / BM, n_fb = (F + BN - 1) / BN;
  const int64_t n_items = (int64_t)d.num_freqs * n_cb * n_fb;
  const int KC = (int)((t_pad + BK - 1) / BK);

  if (tid == 0) {
    for (int i = 0; i < B_STAGES; ++i) {
      mbar_init(&S.b_full[i], 1);
      mbar_init(&S.b_empty[i], 1 + 4);
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
  }
  if (warp == WARP_TMA && lane == 0) {
    tma_prefetch_desc(&map_v);
    tma_prefetch_desc(&map_dhi);
    tma_prefetch_desc(&map_dlo);
  }
  if (warp == WARP_MMA) tmem_alloc<256>(&S.tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = S.tmem_base;

  if (warp == WARP_TMA) {
    uint32_t it = 0;
    for (int64_t w = blockIdx.x; w < n_items; w += gridDim.x) {
      const int fb = (int)(w % n_fb);
      const int cb = (int)((w / n_fb) % n_cb);
      const int q = (int)(w / ((int64_t)n_fb * n_cb));
      for (int kc = 0; kc < KC; ++kc, ++it) {
        const uint32_t s = it % B_STAGES, round = it / B_STAGES;
        mbar_wait(&S.b_empty[s], (round & 1) ^ 1);
        if (elect_one()) {
          mbar_arrive_expect_tx(&S.b_full[s], 4 * VBOX_BYTES + 2 * D_TILE_BYTES);
#pragma unroll
          for (int b = 0; b < 4; ++b) tma_load_3d(S.v[s][b], &map_v, &S.b_full[s], cb * BM + 32 * b, kc * BK, q);
          tma_load_2d(S.d_hi[s], &map_dhi, &S.b_full[s], kc * BK, q * F + fb * BN);
          tma_load_2d(S.d_lo[s], &map_dlo, &S.b_full[s], kc * BK, q * F + fb * BN);
        }
        __syncwarp();
      }
    }
  } else if (warp == WARP_MMA) {
    const uint32_t idesc = idesc_tf32(BM, BN);
    uint32_t it = 0;
    for (int64_t w = blockIdx.x; w < n_items; w += gridDim.x) {
      for (int kc = 0; kc < KC; ++kc, ++it) {
        const uint32_t sb = it % B_STAGES, sa = it % A_STAGES, ab = it % 2;
        const uint64_t dh0 = sdesc_sw128(smem_u32(S.d_hi[sb])), dl0 = sdesc_sw128(smem_u32(S.d_lo[sb]));
        const uint32_t dacc = tmem + COL_ACC + ab * BN;
        mbar_wait(&S.acc_empty[ab], ((it / 2) & 1) ^ 1);
        mbar_wait(&S.a_full[sa], (it / A_STAGES) & 1);
        tc_fence_after();
        const uint32_t a_hi = tmem + COL_A + sa * (2 * BK), a_lo = a_hi + BK;
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < BK / 8; ++k) {
            mma_tf32_ts(dacc, a_hi + 8 * k, dl0 + 2 * k, idesc, k != 0);
            mma_tf32_ts(dacc, a_lo + 8 * k, dh0 + 2 * k, idesc, 1);
          }
#pragma unroll
          for (int k = 0; k < BK / 8; ++k) mma_tf32_ts(dacc, a_hi + 8 * k, dh0 + 2 * k, idesc, 1);
          mma_commit(&S.a_empty[sa]);
          mma_commit(&S.acc_full[ab]);
          mma_commit(&S.b_empty[sb]);
        }
        __syncwarp();
      }
    }
  } else if (warp < 4) {
    const uint32_t lane_addr = tmem + ((uint32_t)(32 * warp) << 16);
    uint32_t it = 0;
    for (int64_t w = blockIdx.x; w < n_items; w += gridDim.x) {
      for (int kc = 0; kc < KC; ++kc, ++it) {
        const uint32_t sb = it % B_STAGES, sa = it % A_STAGES;
        mbar_wait(&S.b_full[sb], (it / B_STAGES) & 1);
        const uint8_t* box = reinterpret_cast<const uint8_t*>(S.v[sb][warp]);
        float hi[BK], lo[BK];
#pragma unroll
        for (int t = 0; t < BK; ++t) {
          const float x = *reinterpret_cast<const float*>(box + sw128_offset(t, lane));
          const float h = __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
          hi[t] = h;
          lo[t] = __fsub_rn(x, h);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&S.b_empty[sb]);
        mbar_wait(&S.a_empty[sa], ((it / A_STAGES) & 1) ^ 1);
        tc_fence_after();
        const uint32_t base = lane_addr + COL_A + sa * (2 * BK);
#pragma unroll
        for (int c = 0; c < BK; c += 16) {
          tmem_st16(base + c, *reinterpret_cast<float(*)[16]>(hi + c));
          tmem_st16(base + BK + c, *reinterpret_cast<float(*)[16]>(lo + c));
        }
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&S.a_full[sa]);
      }
    }
  } else {
    const int quad = warp % 4;
    const int c0 = ((warp - 4) / 4) * EC;
    const uint32_t lane_addr = tmem + ((uint32_t)(32 * quad) << 16);
    uint32_t it = 0;
    for (int64_t w = blockIdx.x; w < n_items; w += gridDim.x) {
      const int fb = (int)(w % n_fb);
      const int cb = (int)((w / n_fb) % n_cb);
      const int q = (int)(w / ((int64_t)n_fb * n_cb));
      float tot[EC], mid[EC];
#pragma unroll
      for (int j = 0; j < EC; ++j) tot[j] = mid[j] = 0.f;
      int nb = 0;
      for (int kc = 0; kc < KC; ++kc, ++it) {
        const uint32_t ab = it % 2;
        mbar_wait(&S.acc_full[ab], (it / 2) & 1);
        tc_fence_after();
        float part[EC];
        tmem_ld32(lane_addr + COL_ACC + ab * BN + c0, part);
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&S.acc_empty[ab]);
        // +1 ulp away from zero: the 4 main-product steps of the chunk each
        // truncate toward zero (dwm_gemm_tc.cu trunc_compensate; an integer
        // add on the float bits)
#pragma unroll
        for (int j = 0; j < EC; ++j) mid[j] = __fadd_rn(mid[j], __uint_as_float(__float_as_uint(part[j]) + 1u));
        if (++nb == BLOCK_CHUNKS) {
          nb = 0;
#pragma unroll
          for (int j = 0; j < EC; ++j) {
            tot[j] = __fadd_rn(tot[j], mid[j]);
            mid[j] = 0.f;
          }
        }
      }
      const int c = cb * BM + 32 * quad + lane;
      if (c < C) {
        float* dst = du + ((int64_t)q * C + c) * F + fb * BN + c0;
#pragma unroll
        for (int j = 0; j < EC; ++j)
          if (fb * BN + c0 + j < F) dst[j] = __fadd_rn(tot[j], mid[j]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == WARP_MMA) tmem_dealloc<256>(tmem);
}

// DM_q[f][t] = (A dY A^T)_q for every part and frequency (plan order, row
// frequency, column frequency -- the V/U order), split into TF32 hi/lo
// planes [q][f][t_pad]; tail t in [tiles, t_pad) written as zeros.
__global__ void grad_out_transform_kernel(const dwm_desc_t d, int64_t t_pad, const float* __restrict__ dy,
                                          float* __restrict__ dhi, float* __restrict__ dlo) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int f = blockIdx.y;
  if (t >= t_pad) return;
  float g[2][2] = {{0.f, 0.f}, {0.f, 0.f}};
  if (t < d.tiles) {
    const int tx = (int)(t % d.tw);
    const int64_t t2 = t / d.tw;
    const int ty = (int)(t2 % d.th);
    const int n = (int)(t2 / d.th);
    const float* src = dy + ((int64_t)n * d.f + f) * d.oh * d.ow;
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int oy = 2 * ty + i, ox = 2 * tx + j;
        if (oy < d.oh && ox < d.ow) g[i][j] = src[(int64_t)oy * d.ow + ox];
      }
  }
  int q = 0;
  for (int rp = 0; rp < d.n_row_parts; ++rp)
    for (int cp = 0; cp < d.n_col_parts; ++cp) {
      const int pr = d.row_parts[rp].count, pc = d.col_parts[cp].count;
      // row stage r[a][j] = sum_i At_r[i][a] g[i][j]; column stage over j
      for (int a = 0; a <= pr; ++a) {
        const float r0 = __fadd_rn(c_at[pr][0][a] * g[0][0], c_at[pr][1][a] * g[1][0]);
        const float r1 = __fadd_rn(c_at[pr][0][a] * g[0][1], c_at[pr][1][a] * g[1][1]);
        for (int b = 0; b <= pc; ++b, ++q) {
          const float v = __fadd_rn(r0 * c_at[pc][0][b], r1 * c_at[pc][1][b]);
          const float hi = tf32_rn(v);
          const int64_t o = ((int64_t)q * d.f + f) * t_pad + t;
          dhi[o] = hi;
          dlo[o] = tf32_rn(v - hi);
        }
      }
    }
}

// gw[f][c][taps of part] = G_r^T dU_part G_c, placed at the part's strided taps.
__global__ void wgrad_place_kernel(const dwm_desc_t d, const float* __restrict__ du, float* __restrict__ gw,
                                   int32_t* __restrict__ flag) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)d.f * d.c) return;
  const int c = (int)(idx % d.c), f = (int)(idx / d.c);
  float* g = gw + idx * d.r_h * d.r_w;
  int q = 0;
  for (int rp = 0; rp < d.n_row_parts; ++rp)
    for (int cp = 0; cp < d.n_col_parts; ++cp) {
      const dwm_axis_part_t R = d.row_parts[rp], Cc = d.col_parts[cp];
      const int pr = R.count, pc = Cc.count, lr = pr + 1, lc = pc + 1;
      float m[4][4];
      for (int a = 0; a < lr; ++a)
        for (int b = 0; b < lc; ++b) m[a][b] = du[((int64_t)(q + a * lc + b) * d.c + c) * d.f + f];
      for (int i = 0; i < pr; ++i)
        for (int j = 0; j < pc; ++j) {
          float acc = 0.f;
          for (int a = 0; a < lr; ++a) {
            float row = 0.f;
            for (int b = 0; b < lc; ++b) row = fmaf(m[a][b], c_g[pc][b][j], row);
            acc = fmaf(c_g[pr][a][i], row, acc);
          }
          g[(R.origin + R.step * i) * d.r_w + Cc.origin + Cc.step * j] = acc;
          if (flag && !isfinite(acc)) *flag = 1;
        }
      q += lr * lc;
    }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult qr;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr) == cudaSuccess &&
        qr == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
  }
  return fn;
}

int encode(CUtensorMap* map, const float* base, int rank, const cuuint64_t* dims, const cuuint64_t* strides,
           const cuuint32_t* box) {
  auto fn = encode_fn();
  if (!fn) return fail(DWM_ECUDA, "cuTensorMapEncodeTiled is unavailable");
  const cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rank, (void*)base, dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(DWM_ECUDA, "cuTensorMapEncodeTiled (weight gradient) failed (%d)", (int)r);
  return DWM_OK;
}

int64_t t_padded(const dwm_desc_t& d) { return (d.tiles + 3) / 4 * 4; }

}  // namespace

bool wgrad_tc_supported(const dwm_desc_t& d) {
  return d.c % 32 == 0 && d.c >= 64 && d.f >= 64 && d.tiles < ((int64_t)1 << 31);
}

size_t wgrad_tc_workspace_bytes(const dwm_desc_t& d) {
  const size_t v = (size_t)d.num_freqs * d.tiles * d.c * 4;
  const size_t dm = 2 * (size_t)d.num_freqs * d.f * t_padded(d) * 4;
  const size_t du = (size_t)d.num_freqs * d.c * d.f * 4;
  return (v + 255) / 256 * 256 + (dm + 255) / 256 * 256 + (du + 255) / 256 * 256;
}

int launch_wgrad_tc(const dwm_desc_t& d, const void* x, const void* dy, void* gw, void* ws, size_t ws_bytes,
                    int32_t* flag, cudaStream_t s) {
  if (!wgrad_tc_supported(d)) return fail(DWM_EUNSUPPORTED, "tcgen05 weight gradient needs C %% 32 == 0, C, F >= 64");
  if (!ws || ws_bytes < wgrad_tc_workspace_bytes(d))
    return fail(DWM_EINVAL_SHAPE, "weight-gradient workspace too small: %zu bytes given, %zu needed", ws_bytes,
                wgrad_tc_workspace_bytes(d));
  const int64_t tp = t_padded(d);
  char* base = (char*)ws;
  float* V = (float*)base;
  base += ((size_t)d.num_freqs * d.tiles * d.c * 4 + 255) / 256 * 256;
  float* dhi = (float*)base;
  float* dlo = dhi + (size_t)d.num_freqs * d.f * tp;
  base += (2 * (size_t)d.num_freqs * d.f * tp * 4 + 255) / 256 * 256;
  float* du = (float*)base;

  if (int st = launch_input_transform(d, DWM_F32, x, V, s)) return st;
  {
    const dim3 grid((unsigned)((tp + 127) / 128), (unsigned)d.f);
    grad_out_transform_kernel<<<grid, 128, 0, s>>>(d, tp, (const float*)dy, dhi, dlo);
    DWM_CUDA_TRY(cudaGetLastError());
  }
  CUtensorMap mv, mh, ml;
  {
    const cuuint64_t dims[3] = {(cuuint64_t)d.c, (cuuint64_t)d.tiles, (cuuint64_t)d.num_freqs};
    const cuuint64_t strides[2] = {(cuuint64_t)d.c * 4, (cuuint64_t)d.tiles * d.c * 4};
    const cuuint32_t box[3] = {32, BK, 1};
    if (int st = encode(&mv, V, 3, dims, strides, box)) return st;
  }
  {
    const cuuint64_t dims[2] = {(cuuint64_t)tp, (cuuint64_t)d.num_freqs * d.f};
    const cuuint64_t strides[1] = {(cuuint64_t)tp * 4};
    const cuuint32_t box[2] = {BK, BN};
    if (int st = encode(&mh, dhi, 2, dims, strides, box)) return st;
    if (int st = encode(&ml, dlo, 2, dims, strides, box)) return st;
  }
  const size_t smem = sizeof(WSmem) + 1024;
  if (int st = ensure_dynamic_smem((const void*)wgrad_tc_kernel, smem)) return st;
  int sms = 0;
  if (int st = device_sm_count(&sms)) return st;
  const int64_t items = (int64_t)d.num_freqs * ((d.c + BM - 1) / BM) * ((d.f + BN - 1) / BN);
  const int grid = (int)(items < sms ? items : sms);
  wgrad_tc_kernel<<<grid, THREADS, smem, s>>>(d, tp, mv, mh, ml, du);
  DWM_CUDA_TRY(cudaGetLastError());
  const int64_t fc = (int64_t)d.f * d.c;
  wgrad_place_kernel<<<(unsigned)((fc + 127) / 128), 128, 0, s>>>(d, du, (float*)gw, flag);
  DWM_CUDA_TRY(cudaGetLastError());
  return DWM_OK;
}

}  // namespace dwm
