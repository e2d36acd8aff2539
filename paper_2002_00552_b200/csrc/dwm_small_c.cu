// dwm_small_c.cu -- fully fused DWM forward for small input-channel counts
// (C_in <= 4: the ResNet-50 / AlexNet stems of BASELINE configs[1], [2]).
//
// With K = C_in <= 4 the per-frequency "GEMM" is not a tensor-core
// contraction (SURVEY §7 hard part 4); the whole forward is FP32-pipe bound.
// One persistent kernel therefore does everything on the CUDA cores and only
// x is read and y written in HBM:
//
//   prologue : U[freq][F][C] (from the filter-transform kernel) -> smem,
//              transposed to [freq][C][f-block] for broadcast float4 reads.
//   per tile block (64 consecutive 2x2 output tiles) and per plan part:
//     producer: polyphase gather of the part's (count+1)^2 input window for
//               every (tile, channel) straight from x (padding and the
//               reference's even-extension zeros by predicate), Bt.d.B row
//               stage then column stage -> V part in smem (double buffered;
//               the x loads of part p+1 are issued before part p's math).
//     consumer: per frequency, M = sum_c U*V (FMA chain, c ascending);
//               At.m.A row stage S, column stage T with compile-time
//               coefficients (0 skipped, +-1 as add/sub); y += T in plan order.
//   epilogue : interleave the 2x2 tiles into NCHW, truncate odd extents,
//              raise the non-finite flag.
//
// Every rounding step is the reference's (engines.py:164-194, 244-255 with a
// sequential BLAS), so the output is bit-identical to the reference DWM in
// binary32 (see tests/test_gpu_parity.py).
#include <utility>

#include "dwm_common.cuh"
#include "dwm_kernels.h"

namespace dwm {
namespace {

constexpr int BM = 64;       // tiles per block
constexpr int BN = 32;       // filters per block
constexpr int TM = 2;        // tiles per thread (strided by 32)
constexpr int TN = 4;        // filters per thread (contiguous)
constexpr int THREADS = 256; // (BM/TM) * (BN/TN)
constexpr int MAXQ = 16;     // frequencies per part, (3+1)^2

// At coefficient of F(2, r): row i (output), column a (frequency).
__host__ __device__ constexpr int at_coef(int r, int i, int a) {
  return r == 1 ? (i == a ? 1 : 0)
       : r == 2 ? (i == 0 ? (a <= 1 ? 1 : 0) : (a == 1 ? 1 : (a == 2 ? -1 : 0)))
                : (i == 0 ? (a <= 2 ? 1 : 0) : (a == 0 ? 0 : (a == 1 ? 1 : -1)));
}

template <int K> __device__ __forceinline__ float cmul(float m) {
  if constexpr (K == 1) return m;
  else if constexpr (K == -1) return -m;
  else return 0.f;
}
// fma(K, m, acc) for K in {0, +-1}: exact skip / add / sub.
template <int K> __device__ __forceinline__ float cfma(float m, float acc) {
  if constexpr (K == 1) return __fadd_rn(acc, m);
  else if constexpr (K == -1) return __fsub_rn(acc, m);
  else return acc;
}

template <typename F, int... Is>
__device__ __forceinline__ void static_for_impl(F&& f, std::integer_sequence<int, Is...>) {
  (f(std::integral_constant<int, Is>{}), ...);
}
template <int N, typename F> __device__ __forceinline__ void static_for(F&& f) {
  static_for_impl(f, std::make_integer_sequence<int, N>{});
}

struct Acc {
  float v[TM][TN][2][2];
};

// Consume one part: sV [q][BM][CC], sU at the part's first frequency [q][CC][BN].
template <int CC, int PR, int PC>
__device__ __forceinline__ void consume_part(const float* __restrict__ sV, const float* __restrict__ sU,
                                             int tm, int tn, Acc& acc, bool first_part) {
  constexpr int LR = PR + 1, LC = PC + 1;
  float T[TM][TN][2][2];
  static_for<LC>([&](auto bI) {
    constexpr int b = decltype(bI)::value;
    float S[TM][TN][2];
    static_for<LR>([&](auto aI) {
      constexpr int a = decltype(aI)::value;
      constexpr int q = a * LC + b;
      float M[TM][TN];
#pragma unroll
      for (int c = 0; c < CC; ++c) {
        float v[TM];
#pragma unroll
        for (int i = 0; i < TM; ++i) v[i] = sV[(q * BM + tm + 32 * i) * CC + c];
        const float4 u4 = *reinterpret_cast<const float4*>(sU + (q * CC + c) * BN + tn * TN);
        const float u[TN] = {u4.x, u4.y, u4.z, u4.w};
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int j = 0; j < TN; ++j)
            M[i][j] = (c == 0) ? __fmul_rn(u[j], v[i]) : __fmaf_rn(u[j], v[i], M[i][j]);
      }
      constexpr int k0 = at_coef(PR, 0, a), k1 = at_coef(PR, 1, a);
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) {
          if constexpr (a == 0) {
            S[i][j][0] = cmul<k0>(M[i][j]);
            S[i][j][1] = cmul<k1>(M[i][j]);
          } else {
            S[i][j][0] = cfma<k0>(M[i][j], S[i][j][0]);
            S[i][j][1] = cfma<k1>(M[i][j], S[i][j][1]);
          }
        }
    });
    constexpr int c0 = at_coef(PC, 0, b), c1 = at_coef(PC, 1, b);
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j)
#pragma unroll
        for (int ii = 0; ii < 2; ++ii) {
          if constexpr (b == 0) {
            T[i][j][ii][0] = cmul<c0>(S[i][j][ii]);
            T[i][j][ii][1] = cmul<c1>(S[i][j][ii]);
          } else {
            T[i][j][ii][0] = cfma<c0>(S[i][j][ii], T[i][j][ii][0]);
            T[i][j][ii][1] = cfma<c1>(S[i][j][ii], T[i][j][ii][1]);
          }
        }
  });
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j)
#pragma unroll
      for (int ii = 0; ii < 2; ++ii)
#pragma unroll
        for (int jj = 0; jj < 2; ++jj)
          acc.v[i][j][ii][jj] = first_part ? T[i][j][ii][jj] : __fadd_rn(acc.v[i][j][ii][jj], T[i][j][ii][jj]);
}

template <int CC>
__device__ __forceinline__ void consume_dispatch(int pr, int pc, const float* sV, const float* sU, int tm,
                                                 int tn, Acc& acc, bool first) {
  switch (pr * 4 + pc) {
    case 5: consume_part<CC, 1, 1>(sV, sU, tm, tn, acc, first); break;
    case 6: consume_part<CC, 1, 2>(sV, sU, tm, tn, acc, first); break;
    case 7: consume_part<CC, 1, 3>(sV, sU, tm, tn, acc, first); break;
    case 9: consume_part<CC, 2, 1>(sV, sU, tm, tn, acc, first); break;
    case 10: consume_part<CC, 2, 2>(sV, sU, tm, tn, acc, first); break;
    case 11: consume_part<CC, 2, 3>(sV, sU, tm, tn, acc, first); break;
    case 13: consume_part<CC, 3, 1>(sV, sU, tm, tn, acc, first); break;
    case 14: consume_part<CC, 3, 2>(sV, sU, tm, tn, acc, first); break;
    default: consume_part<CC, 3, 3>(sV, sU, tm, tn, acc, first); break;
  }
}

// Producer half 1: gather the part's input window for (tile, c) into registers.
__device__ __forceinline__ void load_window(const dwm_desc_t& d, const float* __restrict__ x, int64_t tile,
                                            int c, int rp, int cp, float win[4][4]) {
  const dwm_axis_part_t R = d.row_parts[rp], Cc = d.col_parts[cp];
  const int lr = R.count + 1, lc = Cc.count + 1;
  const int tx = (int)(tile % d.tw);
  const int64_t t2 = tile / d.tw;
  const int ty = (int)(t2 % d.th);
  const int n = (int)(t2 / d.th);
  const bool live = tile < d.tiles;
  const float* xc = x + ((int64_t)n * d.c + c) * d.h * d.w;
  int rows[4], cols[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int k = 2 * ty + i;
    const int row = R.origin + d.s_h * k - d.pad_top;
    rows[i] = (live && i < lr && k < d.oh - 1 + R.count && row >= 0 && row < d.h) ? row : -1;
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int k = 2 * tx + j;
    const int col = Cc.origin + d.s_w * k - d.pad_left;
    cols[j] = (j < lc && k < d.ow - 1 + Cc.count && col >= 0 && col < d.w) ? col : -1;
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
      win[i][j] = (rows[i] >= 0 && cols[j] >= 0) ? __ldg(xc + (int64_t)rows[i] * d.w + cols[j]) : 0.f;
}

// Producer half 2: Bt.d.B (row stage then column stage) -> sV[q][t][c].
template <int CC>
__device__ __forceinline__ void transform_store(const dwm_desc_t& d, int rp, int cp, const float win[4][4],
                                                float* __restrict__ sV, int t, int c) {
  const int pr = d.row_parts[rp].count, pc = d.col_parts[cp].count;
  const int lr = pr + 1, lc = pc + 1;
  float tt[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float acc = __fmul_rn(c_bt[pr][a][0], win[0][j]);
#pragma unroll
      for (int i = 1; i < 4; ++i)
        if (i < lr) acc = __fmaf_rn(c_bt[pr][a][i], win[i][j], acc);
      tt[a][j] = acc;
    }
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
      if (a < lr && b < lc) {
        float acc = __fmul_rn(tt[a][0], c_bt[pc][b][0]);
#pragma unroll
        for (int j = 1; j < 4; ++j)
          if (j < lc) acc = __fmaf_rn(tt[a][j], c_bt[pc][b][j], acc);
        sV[((a * lc + b) * BM + t) * CC + c] = acc;
      }
}

template <int CC>
__global__ void __launch_bounds__(THREADS, 2)
small_c_kernel(const dwm_desc_t d, const float* __restrict__ x, const float* __restrict__ U,
               float* __restrict__ y, int32_t* __restrict__ flag) {
  extern __shared__ __align__(16) float smem[];
  float* sU = smem;                                    // [freq][CC][BN]
  float* sVbuf = smem + (size_t)d.num_freqs * CC * BN; // [2][MAXQ][BM][CC]
  constexpr int VSTAGE = MAXQ * BM * CC;

  const int tid = threadIdx.x;
  const int tm = tid % 32, tn = tid / 32;
  const int f0 = blockIdx.y * BN;
  const int F = d.f;
  const int nparts = d.n_row_parts * d.n_col_parts;
  const int64_t nblocks = (d.tiles + BM - 1) / BM;

  for (int e = tid; e < d.num_freqs * CC * BN; e += THREADS) {
    const int fl = e % BN, c = (e / BN) % CC, q = e / (BN * CC);
    const int f = f0 + fl;
    sU[e] = f < F ? U[((int64_t)q * F + f) * CC + c] : 0.f;
  }

  // producer role: (tile t, channel c) of the block
  const bool producer = tid < BM * CC;
  const int pt = tid / CC, pc_ch = tid % CC;

  int64_t tb = blockIdx.x;
  if (tb >= nblocks) return;
  float win[4][4];
  if (producer) load_window(d, x, tb * BM + pt, pc_ch, 0, 0, win);
  if (producer) transform_store<CC>(d, 0, 0, win, sVbuf, pt, pc_ch);
  __syncthreads();

  int stage = 0;
  Acc acc;
  for (; tb < nblocks; tb += gridDim.x) {
    int qoff = 0;
    for (int p = 0; p < nparts; ++p) {
      const int rp = p / d.n_col_parts, cpi = p % d.n_col_parts;
      // next unit of work: part p+1 of this block, or part 0 of the next block
      const bool has_next = (p + 1 < nparts) || (tb + gridDim.x < nblocks);
      const int np = (p + 1 < nparts) ? p + 1 : 0;
      const int64_t ntb = (p + 1 < nparts) ? tb : tb + gridDim.x;
      const int nrp = np / d.n_col_parts, ncp = np % d.n_col_parts;
      if (producer && has_next) load_window(d, x, ntb * BM + pt, pc_ch, nrp, ncp, win);

      consume_dispatch<CC>(d.row_parts[rp].count, d.col_parts[cpi].count, sVbuf + stage * VSTAGE,
                           sU + qoff * CC * BN, tm, tn, acc, p == 0);
      qoff += (d.row_parts[rp].count + 1) * (d.col_parts[cpi].count + 1);

      if (producer && has_next) transform_store<CC>(d, nrp, ncp, win, sVbuf + (stage ^ 1) * VSTAGE, pt, pc_ch);
      stage ^= 1;
      __syncthreads();
    }
    // epilogue: 2x2 tiles -> NCHW
    bool bad = false;
#pragma unroll
    for (int i = 0; i < TM; ++i) {
      const int64_t tile = tb * BM + tm + 32 * i;
      if (tile >= d.tiles) continue;
      const int tx = (int)(tile % d.tw);
      const int64_t t2 = tile / d.tw;
      const int ty = (int)(t2 % d.th);
      const int n = (int)(t2 / d.th);
#pragma unroll
      for (int j = 0; j < TN; ++j) {
        const int f = f0 + tn * TN + j;
        if (f >= F) continue;
        float* yf = y + ((int64_t)n * F + f) * d.oh * d.ow;
#pragma unroll
        for (int ii = 0; ii < 2; ++ii) {
          const int oy = 2 * ty + ii;
          if (oy >= d.oh) continue;
          const float v0 = acc.v[i][j][ii][0], v1 = acc.v[i][j][ii][1];
          const int ox = 2 * tx;
          float* dst = yf + (int64_t)oy * d.ow + ox;
          if (ox + 1 < d.ow) {
            bad |= !(isfinite(v0) && isfinite(v1));
            if ((d.ow & 1) == 0) {
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
    if (bad && flag) *flag = 1;
  }
}

template <int CC>
int launch_cc(const dwm_desc_t& d, const float* x, const float* U, float* y, int32_t* flag, cudaStream_t s) {
  const size_t smem = ((size_t)d.num_freqs * CC * BN + 2 * (size_t)MAXQ * BM * CC) * sizeof(float);
  DWM_CUDA_TRY(cudaFuncSetAttribute(small_c_kernel<CC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int dev = 0, sms = 0, per_sm = 0;
  DWM_CUDA_TRY(cudaGetDevice(&dev));
  DWM_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  DWM_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, small_c_kernel<CC>, THREADS, smem));
  if (per_sm < 1) return fail(DWM_EUNSUPPORTED, "small-C kernel does not fit (smem %zu B)", smem);
  const int fblocks = (d.f + BN - 1) / BN;
  const int64_t nblocks = (d.tiles + BM - 1) / BM;
  int64_t gx = ((int64_t)sms * per_sm + fblocks - 1) / fblocks;
  if (gx > nblocks) gx = nblocks;
  small_c_kernel<CC><<<dim3((unsigned)gx, (unsigned)fblocks), THREADS, smem, s>>>(d, x, U, y, flag);
  DWM_CUDA_TRY(cudaGetLastError());
  return DWM_OK;
}

}  // namespace

bool small_c_supported(const dwm_desc_t& d) {
  if (d.c < 1 || d.c > 4) return false;
  const size_t smem = ((size_t)d.num_freqs * d.c * BN + 2 * (size_t)MAXQ * BM * d.c) * sizeof(float);
  return smem <= 200 * 1024;
}

int launch_small_c(const dwm_desc_t& d, const void* x, const void* U, void* y, int32_t* flag, cudaStream_t s) {
  const float* xf = (const float*)x;
  const float* Uf = (const float*)U;
  float* yf = (float*)y;
  switch (d.c) {
    case 1: return launch_cc<1>(d, xf, Uf, yf, flag, s);
    case 2: return launch_cc<2>(d, xf, Uf, yf, flag, s);
    case 3: return launch_cc<3>(d, xf, Uf, yf, flag, s);
    case 4: return launch_cc<4>(d, xf, Uf, yf, flag, s);
    default: return fail(DWM_EUNSUPPORTED, "small-C kernel handles C_in <= 4, got %d", d.c);
  }
}

}  // namespace dwm
