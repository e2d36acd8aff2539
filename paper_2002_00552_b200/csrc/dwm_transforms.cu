// dwm_transforms.cu -- filter transform (U = G g Gt) and input-tile transform
// (V = Bt d B with the polyphase stride gather) for every decomposition part.
//
// Reference rows: W (kernel sub-block gather, engines.py:246-248),
// U (engines.py:187), G (strided slice + even zero-extension + windows,
// tensor.py:45-65, engines.py:104-120), V (engines.py:186).
//
// Both transforms apply the row stage then the column stage as sequential
// FMA chains in ascending tap order, so U and V are bit-identical to the
// reference's binary32/binary64 values (the coefficients are 0, +-1, +-1/2).
#include "dwm_common.cuh"
#include "dwm_kernels.h"
#include "dwm_wino.cuh"

#include <cstring>

namespace dwm {

// ---------------------------------------------------------------------------
// Filter transform: one thread per (f, c); U[fq][f][c].
// ---------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ void part_filter_transform(const dwm_desc_t& d, const T* __restrict__ wfc,
                                                      int rp, int cp, T out[4][4]) {
  const dwm_axis_part_t R = d.row_parts[rp], Cc = d.col_parts[cp];
  const int pr = R.count, pc = Cc.count;
  T g[3][3];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      g[i][j] = (i < pr && j < pc) ? wfc[(R.origin + R.step * i) * d.r_w + Cc.origin + Cc.step * j] : T(0);
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

template <typename T>
__global__ void filter_transform_kernel(const dwm_desc_t d, const T* __restrict__ w, T* __restrict__ U) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t fc = (int64_t)d.f * d.c;
  if (idx >= fc) return;
  const T* wfc = w + idx * d.r_h * d.r_w;  // idx = f*C + c
  int fq = 0;
  for (int rp = 0; rp < d.n_row_parts; ++rp)
    for (int cp = 0; cp < d.n_col_parts; ++cp) {
      T u[4][4];
      part_filter_transform(d, wfc, rp, cp, u);
      const int lr = d.row_parts[rp].count + 1, lc = d.col_parts[cp].count + 1;
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b)
          if (a < lr && b < lc) U[(int64_t)(fq + a * lc + b) * fc + idx] = u[a][b];
      fq += lr * lc;
    }
}

__device__ __forceinline__ float tf32_rn(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// U_hi = tf32(U), U_lo = tf32(U - U_hi), two [freq][F][C] planes.
__global__ void filter_transform_tf32split_kernel(const dwm_desc_t d, const float* __restrict__ w,
                                                  float* __restrict__ U) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t fc = (int64_t)d.f * d.c;
  if (idx >= fc) return;
  const int64_t plane = (int64_t)d.num_freqs * fc;
  const float* wfc = w + idx * d.r_h * d.r_w;
  int fq = 0;
  for (int rp = 0; rp < d.n_row_parts; ++rp)
    for (int cp = 0; cp < d.n_col_parts; ++cp) {
      float u[4][4];
      part_filter_transform(d, wfc, rp, cp, u);
      const int lr = d.row_parts[rp].count + 1, lc = d.col_parts[cp].count + 1;
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b)
          if (a < lr && b < lc) {
            const float hi = tf32_rn(u[a][b]);
            const float lo = tf32_rn(u[a][b] - hi);
            const int64_t o = (int64_t)(fq + a * lc + b) * fc + idx;
            U[o] = hi;
            U[plane + o] = lo;
          }
      fq += lr * lc;
    }
}

// ---------------------------------------------------------------------------
// Input transform: one thread per (tile, c), c fastest; V[fq][tile][c].
// Window sample (i, j) of part (rp, cp) for tile (ty, tx) is padded-input
// row a_r + s_h*(2ty+i), col a_c + s_w*(2tx+j)  (decompose.py:117-133), zero
// when it falls in the padding or past the part's strided slice
// (k >= OUT-1+count: the reference's even-extension zeros, engines.py:109-115).
// ---------------------------------------------------------------------------
template <typename T>
__global__ void input_transform_kernel(const dwm_desc_t d, const T* __restrict__ x, T* __restrict__ V) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= d.tiles * d.c) return;
  const int c = (int)(idx % d.c);
  const int64_t tile = idx / d.c;
  const int tx = (int)(tile % d.tw);
  const int64_t t2 = tile / d.tw;
  const int ty = (int)(t2 % d.th);
  const int n = (int)(t2 / d.th);
  const T* xc = x + ((int64_t)n * d.c + c) * d.h * d.w;
  const int64_t tc_stride = d.tiles * d.c;
  int fq = 0;
  for (int rp = 0; rp < d.n_row_parts; ++rp) {
    const dwm_axis_part_t R = d.row_parts[rp];
    const int pr = R.count, lr = pr + 1;
    int rows[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int k = 2 * ty + i;
      const int row = R.origin + d.s_h * k - d.pad_top;
      rows[i] = (i < lr && k < d.oh - 1 + pr && row >= 0 && row < d.h) ? row : -1;
    }
    for (int cp = 0; cp < d.n_col_parts; ++cp) {
      const dwm_axis_part_t Cc = d.col_parts[cp];
      const int pc = Cc.count, lc = pc + 1;
      int cols[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int k = 2 * tx + j;
        const int col = Cc.origin + d.s_w * k - d.pad_left;
        cols[j] = (j < lc && k < d.ow - 1 + pc && col >= 0 && col < d.w) ? col : -1;
      }
      T win[4][4];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
          win[i][j] = (rows[i] >= 0 && cols[j] >= 0) ? __ldg(xc + (int64_t)rows[i] * d.w + cols[j]) : T(0);
      // row stage t[a][j] = sum_i Bt_r[a][i] win[i][j]; column stage v[a][b] = sum_j t[a][j] Bt_c[b][j]
      T t[4][4];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          T acc = mul_rn((T)c_bt[pr][a][0], win[0][j]);
#pragma unroll
          for (int i = 1; i < 4; ++i)
            if (i < lr) acc = fma_rn((T)c_bt[pr][a][i], win[i][j], acc);
          t[a][j] = acc;
        }
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b)
          if (a < lr && b < lc) {
            T acc = mul_rn(t[a][0], (T)c_bt[pc][b][0]);
#pragma unroll
            for (int j = 1; j < 4; ++j)
              if (j < lc) acc = fma_rn(t[a][j], (T)c_bt[pc][b][j], acc);
            V[(int64_t)(fq + a * lc + b) * tc_stride + idx] = acc;
          }
      fq += lr * lc;
    }
  }
}

// ---------------------------------------------------------------------------
// Input transform, shared-memory staged: one CTA per (image, tile row,
// 32-channel block).  The r_h + s_h padded-input rows that tile row reads are
// staged once in shared memory with coalesced row loads; each warp then owns
// tiles, each lane one channel, so every V store is a coalesced 128-byte row
// segment of V[fq][tile][c].  Same arithmetic (and bits) as the kernel above.
// ---------------------------------------------------------------------------
constexpr int IT_CB = 32;  // channels per CTA (one per lane)

// Window gather (compile-time extent, predicated zeros) + Bt.d.B + stores
// to consecutive frequency planes through a running pointer.
template <int PR, int PC, typename T>
__device__ __forceinline__ void it_gather_part(const T* __restrict__ sc, const int (&rows)[4], const int (&cols)[4],
                                               T* vq, int64_t stride) {
  T win[4][4];
#pragma unroll
  for (int i = 0; i <= PR; ++i)
#pragma unroll
    for (int j = 0; j <= PC; ++j) win[i][j] = (rows[i] >= 0 && cols[j] >= 0) ? sc[rows[i] + cols[j]] : T(0);
  wino::input_transform_part<PR, PC>(win, [&](int, T v) {
    *vq = v;
    vq += stride;
  });
}

template <typename T>
__global__ void __launch_bounds__(256)
input_transform_smem_kernel(const dwm_desc_t d, const T* __restrict__ x, T* __restrict__ V, int rows_staged) {
  extern __shared__ __align__(16) unsigned char it_smem_raw[];
  T* sx = reinterpret_cast<T*>(it_smem_raw);  // [IT_CB][rows_staged][W] with odd channel pitch
  const int pitch = rows_staged * d.w + 1;
  // channel block fastest: the C/32 CTAs of one tile row run together
  const int ty = blockIdx.y % d.th;
  const int n = blockIdx.y / d.th;
  const int c0 = blockIdx.x * IT_CB;
  const int cb = min(IT_CB, d.c - c0);
  const int row0 = 2 * ty * d.s_h - d.pad_top;  // padded-input row of window sample 0 (origin 0)

  // stage rows row0 .. row0 + rows_staged - 1 (zero outside [0, H))
  constexpr int VEC = 16 / sizeof(T);
  constexpr int SLOTS = 4;  // (row, vector) slots per lane: up to 128 float4 per channel row block
  if (d.w % VEC == 0 && rows_staged * (d.w / VEC) <= 32 * SLOTS) {
    // 16-byte loads; each lane owns fixed (row, vector) slots of the staged block
    const int wv = d.w / VEC, nslots = rows_staged * wv;
    const int lane = threadIdx.x % 32;
    int srow[SLOTS], scol[SLOTS];
#pragma unroll
    for (int k = 0; k < SLOTS; ++k) {
      const int p = lane + 32 * k;
      srow[k] = p < nslots ? p / wv : -1;
      scol[k] = p < nslots ? (p % wv) * VEC : 0;
    }
    for (int cc = threadIdx.x / 32; cc < cb; cc += blockDim.x / 32) {
      const T* xc = x + ((int64_t)n * d.c + c0 + cc) * d.h * d.w;
      T* dst = sx + cc * pitch;
#pragma unroll
      for (int k = 0; k < SLOTS; ++k) {
        if (srow[k] < 0) continue;
        const int row = row0 + srow[k];
        T v[VEC];
        if (row >= 0 && row < d.h) {
          const float4 q = __ldg(reinterpret_cast<const float4*>(xc + (int64_t)row * d.w + scol[k]));
          memcpy(v, &q, 16);
        } else {
#pragma unroll
          for (int e = 0; e < VEC; ++e) v[e] = T(0);
        }
#pragma unroll
        for (int e = 0; e < VEC; ++e) dst[srow[k] * d.w + scol[k] + e] = v[e];
      }
    }
  } else {
    for (int cc = threadIdx.x / 32; cc < cb; cc += blockDim.x / 32) {
      const T* xc = x + ((int64_t)n * d.c + c0 + cc) * d.h * d.w;
      T* dst = sx + cc * pitch;
      for (int r = 0; r < rows_staged; ++r) {
        const int row = row0 + r;
        if (row >= 0 && row < d.h) {
          const T* src = xc + (int64_t)row * d.w;
          for (int col = threadIdx.x % 32; col < d.w; col += 32) dst[r * d.w + col] = __ldg(src + col);
        } else {
          for (int col = threadIdx.x % 32; col < d.w; col += 32) dst[r * d.w + col] = T(0);
        }
      }
    }
  }
  __syncthreads();

  const int lane = threadIdx.x % 32, warp = threadIdx.x / 32, nwarps = blockDim.x / 32;
  if (lane >= cb) return;
  const T* sc = sx + lane * pitch;
  const int64_t tc_stride = d.tiles * d.c;
  for (int tx = warp; tx < d.tw; tx += nwarps) {
    const int64_t tile = ((int64_t)n * d.th + ty) * d.tw + tx;
    T* vout = V + tile * d.c + c0 + lane;
    int fq = 0;
    for (int rp = 0; rp < d.n_row_parts; ++rp) {
      const dwm_axis_part_t R = d.row_parts[rp];
      const int pr = R.count, lr = pr + 1;
      int rows[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int k = 2 * ty + i;
        const int rs = R.origin + d.s_h * i;  // staged-row index
        const int row = row0 + rs;
        rows[i] = (i < lr && k < d.oh - 1 + pr && row >= 0 && row < d.h) ? rs * d.w : -1;
      }
      for (int cp = 0; cp < d.n_col_parts; ++cp) {
        const dwm_axis_part_t Cc = d.col_parts[cp];
        const int pc = Cc.count, lc = pc + 1;
        int cols[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int k = 2 * tx + j;
          const int col = Cc.origin + d.s_w * k - d.pad_left;
          cols[j] = (j < lc && k < d.ow - 1 + pc && col >= 0 && col < d.w) ? col : -1;
        }
        T* vq = vout + (int64_t)fq * tc_stride;
#define DWM_ITP(A, B) it_gather_part<A, B>(sc, rows, cols, vq, tc_stride)
        DWM_PART_SWITCH(pr, pc, DWM_ITP)
#undef DWM_ITP
        fq += lr * lc;
      }
    }
  }
}

static inline unsigned grid_for(int64_t n, int block) { return (unsigned)((n + block - 1) / block); }

int launch_filter_transform(const dwm_desc_t& d, int dtype, const void* w, void* U, cudaStream_t s) {
  const int64_t n = (int64_t)d.f * d.c;
  if (dtype == DWM_F64)
    filter_transform_kernel<double><<<grid_for(n, 128), 128, 0, s>>>(d, (const double*)w, (double*)U);
  else
    filter_transform_kernel<float><<<grid_for(n, 128), 128, 0, s>>>(d, (const float*)w, (float*)U);
  DWM_CUDA_TRY(cudaGetLastError());
  return DWM_OK;
}

int launch_filter_transform_tf32split(const dwm_desc_t& d, const void* w, void* U, cudaStream_t s) {
  const int64_t n = (int64_t)d.f * d.c;
  filter_transform_tf32split_kernel<<<grid_for(n, 128), 128, 0, s>>>(d, (const float*)w, (float*)U);
  DWM_CUDA_TRY(cudaGetLastError());
  return DWM_OK;
}

template <typename T>
static int launch_input_smem(const dwm_desc_t& d, const void* x, void* V, cudaStream_t s, bool* used) {
  // rows a tile row reads: (largest tap origin + s*count) over row parts = r_h + s_h - 1, +1
  int rows = 0;
  for (int i = 0; i < d.n_row_parts; ++i)
    rows = max(rows, d.row_parts[i].origin + d.s_h * d.row_parts[i].count + 1);
  const size_t smem = (size_t)IT_CB * ((size_t)rows * d.w + 1) * sizeof(T);
  *used = false;
  if (smem > 96 * 1024 || d.c < 8) return DWM_OK;
  DWM_CUDA_TRY(cudaFuncSetAttribute(input_transform_smem_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem));
  const dim3 grid((unsigned)((d.c + IT_CB - 1) / IT_CB), (unsigned)((int64_t)d.n * d.th));
  // warps: a divisor of the tile-row length in [4, 8] so every warp gets the same number of tiles
  int warps = 8;
  if (d.tw <= 8) warps = d.tw;
  else
    for (int cand = 8; cand >= 4; --cand)
      if (d.tw % cand == 0) { warps = cand; break; }
  input_transform_smem_kernel<T><<<grid, 32 * warps, smem, s>>>(d, (const T*)x, (T*)V, rows);
  DWM_CUDA_TRY(cudaGetLastError());
  *used = true;
  return DWM_OK;
}

int launch_input_transform(const dwm_desc_t& d, int dtype, const void* x, void* V, cudaStream_t s) {
  bool used = false;
  const int st = dtype == DWM_F64 ? launch_input_smem<double>(d, x, V, s, &used)
                                  : launch_input_smem<float>(d, x, V, s, &used);
  if (st || used) return st;
  const int64_t n = d.tiles * d.c;
  if (dtype == DWM_F64)
    input_transform_kernel<double><<<grid_for(n, 256), 256, 0, s>>>(d, (const double*)x, (double*)V);
  else
    input_transform_kernel<float><<<grid_for(n, 256), 256, 0, s>>>(d, (const float*)x, (float*)V);
  DWM_CUDA_TRY(cudaGetLastError());
  return DWM_OK;
}

}  // namespace dwm

namespace dwm {

// ---------------------------------------------------------------------------
// Weight gradient: dW[f,c,ky,kx] = sum_{n,oy,ox}
// dY[n,f,oy,ox] * x_pad[n,c,s_h*oy+ky,s_w*ox+kx].  One warp per (f, c, ky):
// lanes stride over (n, oy, ox) in a fixed order, kx taps in registers, then a
// fixed-order warp-shuffle reduction -- deterministic run to run.
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(256) weight_grad_kernel(const dwm_desc_t d, const T* __restrict__ x,
                                                          const T* __restrict__ dy, T* __restrict__ gw) {
  const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x % 32;
  const int64_t nw = (int64_t)d.f * d.c * d.r_h;
  if (wid >= nw) return;
  const int ky = (int)(wid % d.r_h);
  const int c = (int)((wid / d.r_h) % d.c);
  const int f = (int)(wid / ((int64_t)d.r_h * d.c));
  constexpr int MAXR = 16;
  T acc[MAXR];
#pragma unroll
  for (int k = 0; k < MAXR; ++k) acc[k] = T(0);
  const int64_t per_img = (int64_t)d.oh * d.ow;
  const int64_t total = (int64_t)d.n * per_img;
  for (int64_t e = lane; e < total; e += 32) {
    const int n = (int)(e / per_img);
    const int rem = (int)(e % per_img);
    const int oy = rem / d.ow, ox = rem % d.ow;
    const T g = dy[(((int64_t)n * d.f + f) * d.oh + oy) * d.ow + ox];
    const int row = d.s_h * oy + ky - d.pad_top;
    if (row < 0 || row >= d.h) continue;
    const T* xr = x + (((int64_t)n * d.c + c) * d.h + row) * d.w;
    const int col0 = d.s_w * ox - d.pad_left;
#pragma unroll
    for (int kx = 0; kx < MAXR; ++kx) {
      if (kx >= d.r_w) break;
      const int col = col0 + kx;
      if (col >= 0 && col < d.w) acc[kx] = fma_rn(g, xr[col], acc[kx]);
    }
  }
#pragma unroll
  for (int kx = 0; kx < MAXR; ++kx) {
    if (kx >= d.r_w) break;
    T v = acc[kx];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v = add_rn(v, __shfl_xor_sync(0xffffffffu, v, off));
    if (lane == 0) gw[((((int64_t)f * d.c + c) * d.r_h) + ky) * d.r_w + kx] = v;
  }
}

int launch_weight_grad(const dwm_desc_t& d, int dtype, const void* x, const void* dy, void* gw, cudaStream_t s) {
  if (d.r_w > 16) return fail(DWM_EUNSUPPORTED, "weight gradient kernel supports r_w <= 16, got %d", d.r_w);
  const int64_t warps = (int64_t)d.f * d.c * d.r_h;
  const unsigned grid = (unsigned)((warps * 32 + 255) / 256);
  if (dtype == DWM_F64)
    weight_grad_kernel<double><<<grid, 256, 0, s>>>(d, (const double*)x, (const double*)dy, (double*)gw);
  else
    weight_grad_kernel<float><<<grid, 256, 0, s>>>(d, (const float*)x, (const float*)dy, (float*)gw);
  DWM_CUDA_TRY(cudaGetLastError());
  return DWM_OK;
}

}  // namespace dwm
