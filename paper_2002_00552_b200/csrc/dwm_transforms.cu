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
#include "dwm_filter.cuh"
#include "dwm_wino.cuh"

#include <algorithm>
#include <cstdlib>
#include <cstring>

namespace dwm {

// ---------------------------------------------------------------------------
// Filter transform: one thread per (f, c); U[fq][f][c].
// ---------------------------------------------------------------------------
template <typename T>
__global__ void filter_transform_kernel(const dwm_desc_t d, const T* __restrict__ w, const FiltView fv,
                                        T* __restrict__ U) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t fc = (int64_t)d.f * d.c;
  if (idx >= fc) return;
  const T* wfc = w + (idx / d.c) * fv.sf + (idx % d.c) * fv.sc;  // idx = f*C + c
  int fq = 0;
  for (int rp = 0; rp < d.n_row_parts; ++rp)
    for (int cp = 0; cp < d.n_col_parts; ++cp) {
      T u[4][4];
      part_filter_transform(d, wfc, fv, rp, cp, u);
      const int lr = d.row_parts[rp].count + 1, lc = d.col_parts[cp].count + 1;
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b)
          if (a < lr && b < lc) U[(int64_t)(fq + a * lc + b) * fc + idx] = u[a][b];
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
__global__ void input_transform_kernel(const dwm_desc_t d, const T* __restrict__ x, T* __restrict__ V,
                                       uint32_t* __restrict__ xmax) {
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
  float amax = 0.f;
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
      if (xmax) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) amax = fmaxf(amax, fabsf((float)win[i][j]));
      }
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
  if (xmax) atomicMax(xmax + n, __float_as_uint(amax));  // (fallback kernel: lanes may span images)
}

// ---------------------------------------------------------------------------
// Input transform, shared-memory staged: one CTA per (image, tile row,
// 32-channel block).  The r_h + s_h padded-input rows that tile row reads are
// staged once in shared memory with coalesced row loads; each warp then owns
// tiles, each lane one channel, so every V store is a coalesced 128-byte row
// segment of V[fq][tile][c].  Same arithmetic (and bits) as the kernel above.
// ---------------------------------------------------------------------------

#ifndef DWM_IT_TROWS
#define DWM_IT_TROWS 4  // tile rows per CTA (whole-row staging, few-frequency plans)
#endif
// Measured: 4 tile rows per CTA take cfg4 3x3 from
// 0.452 to 0.411 ms; every plan with more frequencies got slower with 2 or 4
// (7x7: +14 %, cfg5 3x3/2: +3 %), so only single-part F(2,<=3) plans use it.
constexpr int IT_TROWS_MAX_FREQS = 16;
constexpr int IT_STREAM_MIN_FREQS = 64;  // evict-first V stores above this many frequencies

// Window gather (compile-time extent, predicated zeros) + Bt.d.B + stores
// to consecutive frequency planes through a running pointer.  STREAM: V
// stores with the evict-first hint (st.global.cs) -- measured faster for the
// many-frequency plans (V/x >= 25: cfg4 7x7 -9 %, 11x11 -7 %), slower for
// 3x3 (+4 %: there the staged-row overlap between neighbouring tile rows is
// re-read from L2), see DESIGN.md section 3.3.
// CSTR = compile-time column stride s_w (1 or 2; 0 = runtime), no CHECK: one
// row pointer per window row and immediate column offsets instead of an
// address add per sample.
template <int PR, int PC, bool CHECK, bool STREAM, int CSTR, typename T>
__device__ __forceinline__ void it_gather_part(const T* __restrict__ sc, const int (&rows)[4], const int (&cols)[4],
                                               T* vq, int64_t stride) {
  // the staged block is zero-padded, so only the even-extension truncation
  // at an odd last tile row / column needs a predicate (CHECK)
  T win[4][4];
#pragma unroll
  for (int i = 0; i <= PR; ++i) {
    if constexpr (CSTR > 0 && !CHECK) {
      const T* r = sc + rows[i] + cols[0];
#pragma unroll
      for (int j = 0; j <= PC; ++j) win[i][j] = r[CSTR * j];
    } else {
#pragma unroll
      for (int j = 0; j <= PC; ++j)
        win[i][j] = (!CHECK || (rows[i] >= 0 && cols[j] >= 0)) ? sc[rows[i] + cols[j]] : T(0);
    }
  }
  wino::input_transform_part<PR, PC>(win, [&](int, T v) {
    if constexpr (STREAM) __stcs(vq, v);
    else *vq = v;
    vq += stride;
  });
}

// Division by a per-launch constant with a host-computed magic number
// (q = (umulhi(n, m) + n) >> s, exact for 0 <= n < 2^31): the staging loop's
// (channel, row, vector) decomposition ran on emulated integer division
// (IABS/I2F/MUFU.RCP sequences were ~30 % of the kernel's instructions on cfg5).
struct FastDiv {
  uint32_t d, m, s;
};
static FastDiv make_fastdiv(uint32_t d) {
  FastDiv f{d, 0, 0};
  while ((1u << f.s) < d) ++f.s;
  f.m = (uint32_t)((((uint64_t)1 << 32) * (((uint64_t)1 << f.s) - d)) / d + 1);
  return f;
}
__device__ __forceinline__ int fdiv(int n, const FastDiv& f) {
  return (int)((__umulhi((uint32_t)n, f.m) + (uint32_t)n) >> f.s);
}
struct ItDivs {
  FastDiv nslots, wv, rpad, npad, nty;  // rows_staged*W/VEC, W/VEC, rows_staged*npad, npad, tile-row groups
};

// byte offset of the gather tables in the input transform's dynamic smem
template <typename T>
__host__ __device__ __forceinline__ size_t it_tab_offset(int cb, int pitch) {
  return ((size_t)cb * pitch * sizeof(T) + 15) & ~(size_t)15;
}
__host__ __device__ __forceinline__ size_t it_tab_bytes(const dwm_desc_t& d, int twl, int trows) {
  return (((size_t)d.n_col_parts * twl * 8 + 15) & ~(size_t)15) + (size_t)trows * d.n_row_parts * 16;
}

#ifndef DWM_IT_MAXNREG
#define DWM_IT_MAXNREG 56  // 5 CTAs of 224 threads per SM (tools/it_exp.sh); binary64 spills a little
#endif
// CB: channels per CTA.  32 (one per lane, every V store a 128-byte row
// segment) or 16 (two tiles per warp step, 64-byte segments; half the staged
// rows per CTA, so twice the resident CTAs on the stride-2 plans whose
// staged block is large).
template <typename T, bool WIDE, bool STREAM, int CB>
__global__ void __maxnreg__(DWM_IT_MAXNREG)
input_transform_smem_kernel(const dwm_desc_t d, const T* __restrict__ x, T* __restrict__ V, int rows_staged,
                            int twb_arg, int ws_arg, int trows_arg, int n0, uint32_t* __restrict__ xmax,
                            const ItDivs dv) {
  // WIDE == false: whole rows staged (ws == W, trows tile rows per CTA) -- the
  // common case, compiled without any of the column-block arithmetic
  const int twb = WIDE ? twb_arg : d.tw;
  const int trows = WIDE ? 1 : trows_arg;  // tile rows per CTA (their staged rows overlap)
  const int ws = WIDE ? ws_arg : d.pad_left + d.w + d.pad_right;  // staged row width (zero-padded)
  extern __shared__ __align__(16) unsigned char it_smem_raw[];
  __shared__ uint32_t s_amax, s_arrived;  // CTA-level max|x| (one global atomic per CTA)
  if (threadIdx.x == 0) s_amax = 0, s_arrived = 0;  // ordered by the __syncthreads after staging
  T* sx = reinterpret_cast<T*>(it_smem_raw);  // [CB][rows_staged][ws] with odd channel pitch
  const int pitch = rows_staged * ws + 1;
  // channel block fastest: the C/32 CTAs of one tile row (segment) run together.
  // Wide images: a CTA covers tiles [tx0, tx0 + twb) of the row and stages only
  // the ws input columns they read (ws == W, tx0 == 0 when the row fits).
  const int nxb = WIDE ? (d.tw + twb - 1) / twb : 1;
  const int tx0 = WIDE ? (int)(blockIdx.y % nxb) * twb : 0;
  const int nty = WIDE ? d.th : (d.th + trows - 1) / trows;
  // magic-number divisions in the non-streaming variants only: the streaming
  // (many-frequency) ones measured 2-5 % slower with them (profiles/r2/ab_it_fastdiv.txt)
  constexpr bool FD = !STREAM;
  const int by_n = WIDE ? 0 : (FD ? fdiv((int)blockIdx.y, dv.nty) : (int)blockIdx.y / nty);  // image (whole-row CTAs)
  const int ty0 = WIDE ? (int)(blockIdx.y / nxb) % d.th : ((int)blockIdx.y - by_n * nty) * trows;
  const int n = n0 + (WIDE ? (int)(blockIdx.y / (nxb * d.th)) : by_n);
  const int cbase = WIDE ? 2 * tx0 * d.s_w - d.pad_left : -d.pad_left;  // input column of staged column 0
  const int c0 = blockIdx.x * CB;
  const int cb = min(CB, d.c - c0);
  const int row0 = 2 * ty0 * d.s_h - d.pad_top;  // padded-input row of window sample 0 (origin 0)

  // stage rows row0 .. row0 + rows_staged - 1 (zero outside [0, H))
  constexpr int VEC = 16 / sizeof(T);
  float amax = 0.f;  // max|x| staged (float path; NaN-blind -- NaN reaches V and the flag anyway)
  if (!WIDE && d.w % VEC == 0 && ((uintptr_t)x & 15) == 0) {
    // 16-byte loads over the flattened (channel, row, vector) space, four per
    // thread in flight before the first smem store waits on one
    const int wv = d.w / VEC, nslots = rows_staged * wv, nitems = cb * nslots;
    const int npad = d.pad_left + d.pad_right;
    for (int p = threadIdx.x; p < cb * rows_staged * npad; p += blockDim.x) {
      const int cc = FD ? fdiv(p, dv.rpad) : p / (rows_staged * npad), rz = p - cc * rows_staged * npad;
      const int r = FD ? fdiv(rz, dv.npad) : rz / npad, z = rz - r * npad;
      sx[cc * pitch + r * ws + (z < d.pad_left ? z : d.w + z)] = T(0);
    }
#ifndef DWM_IT_LOADS
#define DWM_IT_LOADS 4
#endif
    constexpr int U = DWM_IT_LOADS;
    for (int p0 = threadIdx.x; p0 < nitems; p0 += U * blockDim.x) {
      float4 q[U];
      int dsto[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int p = p0 + u * blockDim.x;
        const int cc = FD ? fdiv(p, dv.nslots) : p / nslots, rs = p - cc * nslots;
        const int sr = FD ? fdiv(rs, dv.wv) : rs / wv, scv = (rs - sr * wv) * VEC;
        const int row = row0 + sr;
        const bool ok = p < nitems && row >= 0 && row < d.h;
        q[u] = ok ? __ldg(reinterpret_cast<const float4*>(x + (((int64_t)n * d.c + c0 + cc) * d.h + row) * d.w + scv))
                  : make_float4(0.f, 0.f, 0.f, 0.f);
        dsto[u] = p < nitems ? cc * pitch + sr * ws + d.pad_left + scv : -1;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (dsto[u] < 0) break;
        T v[VEC];
        memcpy(v, &q[u], 16);
#pragma unroll
        for (int e = 0; e < VEC; ++e) sx[dsto[u] + e] = v[e];
        if constexpr (sizeof(T) == 4) {
#pragma unroll
          for (int e = 0; e < VEC; ++e) amax = fmaxf(amax, fabsf((float)v[e]));
        }
      }
    }
  } else {
    for (int cc = threadIdx.x / 32; cc < cb; cc += blockDim.x / 32) {
      const T* xc = x + ((int64_t)n * d.c + c0 + cc) * d.h * d.w;
      T* dst = sx + cc * pitch;
      for (int r = 0; r < rows_staged; ++r) {
        const int row = row0 + r;
        const bool rok = row >= 0 && row < d.h;
        const T* src = xc + (int64_t)(rok ? row : 0) * d.w;
        for (int sc = threadIdx.x % 32; sc < ws; sc += 32) {
          const int col = cbase + sc;
          const T v = (rok && col >= 0 && col < d.w) ? __ldg(src + col) : T(0);
          dst[r * ws + sc] = v;
          if constexpr (sizeof(T) == 4) amax = fmaxf(amax, fabsf((float)v));
        }
      }
    }
  }
  // Gather offset tables (after the staged block): the staged-column offsets
  // of the 4 window columns per (column part, tile column) and the
  // staged-row offsets per (tile row, row part), -1 where the even extension
  // truncates.  The values are the same for every channel lane, so the
  // gather reads them (one broadcast LDS) instead of recomputing the
  // predicates per tile and part (~30 % of the instructions on cfg5).
  // (non-streaming variants only: the streaming ones measured slower with any
  // change to this code, profiles/r2/ab_it_tables.txt)
  constexpr bool TAB = !STREAM;
  const int ncp = d.n_col_parts, nrp = d.n_row_parts;
  const int twl = WIDE ? twb : d.tw;
  short4* colsT = reinterpret_cast<short4*>(it_smem_raw + it_tab_offset<T>(CB, pitch));
  int4* rowsT = reinterpret_cast<int4*>(it_smem_raw + it_tab_offset<T>(CB, pitch) + (((size_t)ncp * twl * 8 + 15) & ~(size_t)15));
  for (int e = threadIdx.x; TAB && e < ncp * twl; e += blockDim.x) {
    const int cp = e / twl, tx = tx0 + (e - cp * twl);
    const dwm_axis_part_t Cc = d.col_parts[cp];
    const int pc = Cc.count, lc = pc + 1;
    short c[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int k = 2 * tx + j;
      const int col = Cc.origin + d.s_w * k - d.pad_left;  // staged columns cover every col read
      c[j] = (short)((j < lc && k < d.ow - 1 + pc) ? col - cbase : -1);
    }
    colsT[e] = make_short4(c[0], c[1], c[2], c[3]);
  }
  for (int e = threadIdx.x; TAB && e < trows * nrp; e += blockDim.x) {
    const int tyl = e / nrp, rp = e - tyl * nrp, ty = ty0 + tyl;
    const dwm_axis_part_t R = d.row_parts[rp];
    const int pr = R.count, lr = pr + 1;
    int r[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int k = 2 * ty + i;
      const int rs = R.origin + d.s_h * (i + 2 * tyl);  // staged-row index (rows outside x are staged zeros)
      r[i] = (i < lr && k < d.oh - 1 + pr) ? rs * ws : -1;
    }
    rowsT[e] = make_int4(r[0], r[1], r[2], r[3]);
  }
  __syncthreads();
  if (xmax) {
    // per warp into shared memory, the CTA's last warp into the image's slot:
    // one global atomic per CTA (per-warp global atomics on the image's one
    // address serialised in L2: cfg4 5x5 input transform 1.00 -> 1.16 ms)
    const uint32_t m = __reduce_max_sync(0xffffffffu, __float_as_uint(amax));
    if (threadIdx.x % 32 == 0) {
      atomicMax(&s_amax, m);
      __threadfence_block();
      if (atomicAdd(&s_arrived, 1u) == blockDim.x / 32 - 1) atomicMax(xmax + n, atomicMax(&s_amax, 0u));
    }
  }

  constexpr int TPW = 32 / CB;  // tiles per warp step
  const int lane = threadIdx.x % 32, warp = threadIdx.x / 32, nwarps = blockDim.x / 32;
  const int cl = lane % CB, sub = lane / CB;
  if (cl >= cb) return;
  const T* sc = sx + cl * pitch;
  const int64_t tc_stride = d.tiles * d.c;
  const int tx_end = WIDE ? min(d.tw, tx0 + twb) : d.tw;
  const int ntr = min(trows, d.th - ty0);
  for (int tyl = 0; tyl < ntr; ++tyl)
  for (int tx = tx0 + warp * TPW + sub; tx < tx_end; tx += nwarps * TPW) {
    const int ty = ty0 + tyl;
    const int64_t tile = ((int64_t)n * d.th + ty) * d.tw + tx;
    T* vout = V + tile * d.c + c0 + cl;
    int fq = 0;
    // even-extension truncation only reaches an odd last tile row / column
    const bool check = 2 * ty >= d.oh - 1 || 2 * tx >= d.ow - 1;
    for (int rp = 0; rp < nrp; ++rp) {
      const dwm_axis_part_t R = d.row_parts[rp];
      const int pr = R.count, lr = pr + 1;
      int rows[4];
      if constexpr (TAB) {
        const int4 r4 = rowsT[tyl * nrp + rp];
        rows[0] = r4.x, rows[1] = r4.y, rows[2] = r4.z, rows[3] = r4.w;
      } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int k = 2 * ty + i;
          const int rs = R.origin + d.s_h * (i + 2 * tyl);  // staged-row index (rows outside x are staged zeros)
          rows[i] = (i < lr && k < d.oh - 1 + pr) ? rs * ws : -1;
        }
      }
      for (int cp = 0; cp < ncp; ++cp) {
        const dwm_axis_part_t Cc = d.col_parts[cp];
        const int pc = Cc.count, lc = pc + 1;
        int cols[4];
        if constexpr (TAB) {
          const short4 c4 = colsT[cp * twl + (tx - tx0)];
          cols[0] = c4.x, cols[1] = c4.y, cols[2] = c4.z, cols[3] = c4.w;
        } else {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int k = 2 * tx + j;
            const int col = Cc.origin + d.s_w * k - d.pad_left;  // staged columns cover every col read
            cols[j] = (j < lc && k < d.ow - 1 + pc) ? col - cbase : -1;
          }
        }
        T* vq = vout + (int64_t)fq * tc_stride;
        if (check) {
#define DWM_ITP(A, B) it_gather_part<A, B, true, STREAM, 0>(sc, rows, cols, vq, tc_stride)
          DWM_PART_SWITCH(pr, pc, DWM_ITP)
#undef DWM_ITP
        } else {
#define DWM_ITP(A, B) it_gather_part<A, B, false, STREAM, 0>(sc, rows, cols, vq, tc_stride)
#define DWM_ITPU(A, B) it_gather_part<A, B, false, STREAM, 1>(sc, rows, cols, vq, tc_stride)
#define DWM_ITP2(A, B) it_gather_part<A, B, false, STREAM, 2>(sc, rows, cols, vq, tc_stride)
          if (d.s_w == 1) {
            DWM_PART_SWITCH(pr, pc, DWM_ITPU)
          } else if (d.s_w == 2) {
            DWM_PART_SWITCH(pr, pc, DWM_ITP2)
          } else {
            DWM_PART_SWITCH(pr, pc, DWM_ITP)
          }
#undef DWM_ITP2
#undef DWM_ITPU
#undef DWM_ITP
        }
        fq += lr * lc;
      }
    }
  }
}

// 16-channel input-transform CTAs: only for strided plans whose 32-channel
// staged block is large (cfg5 5x5/2: 54 KB -> 4 resident CTAs; with 16
// channels 5: 1.58 -> 1.48 ms); every other BASELINE shape was slower
// (cfg4 11x11 +30 %, cfg5 3x3/2 +16 %; profiles/r2/ab_it_cb16.txt).
static bool it_prefers_cb16(const dwm_desc_t& d) {
  if (d.s_h < 2 && d.s_w < 2) return false;
  int rows = 0;
  for (int i = 0; i < d.n_row_parts; ++i)
    rows = max(rows, d.row_parts[i].origin + d.s_h * d.row_parts[i].count + 1);
  const size_t smem32 = (size_t)32 * ((size_t)rows * (d.pad_left + d.w + d.pad_right) + 1) * sizeof(float);
  return smem32 > 48 * 1024;
}

static inline unsigned grid_for(int64_t n, int block) { return (unsigned)((n + block - 1) / block); }

int launch_filter_transform(const dwm_desc_t& d, int dtype, const void* w, void* U, cudaStream_t s,
                            const int64_t* strides) {
  const int64_t n = (int64_t)d.f * d.c;
  const FiltView fv = strides ? FiltView{strides[0], strides[1], strides[2], strides[3]} : contiguous_view(d);
  if (dtype == DWM_F64)
    filter_transform_kernel<double><<<grid_for(n, 128), 128, 0, s>>>(d, (const double*)w, fv, (double*)U);
  else
    filter_transform_kernel<float><<<grid_for(n, 128), 128, 0, s>>>(d, (const float*)w, fv, (float*)U);
  DWM_CUDA_TRY(cudaGetLastError());
  return DWM_OK;
}

template <typename T, int CB>
static int launch_input_smem_cb(const dwm_desc_t& d, const void* x, void* V, cudaStream_t s, bool* used,
                                uint32_t* xmax) {
  // rows a tile row reads: (largest tap origin + s*count) over row parts = r_h + s_h - 1, +1
  int rows = 0;
  for (int i = 0; i < d.n_row_parts; ++i)
    rows = max(rows, d.row_parts[i].origin + d.s_h * d.row_parts[i].count + 1);
  // columns the tiles [tx0, tx0 + twb) read: 2*s_w*(twb-1) + max(origin + s_w*count) + 1
  int cols1 = 0;
  for (int i = 0; i < d.n_col_parts; ++i)
    cols1 = max(cols1, d.col_parts[i].origin + d.s_w * d.col_parts[i].count + 1);
  *used = false;
  if (d.c < 8) return DWM_OK;
  constexpr size_t CAP = 96 * 1024;
  int twb = d.tw, ws = d.pad_left + d.w + d.pad_right;  // whole zero-padded rows
  size_t smem = (size_t)CB * ((size_t)rows * ws + 1) * sizeof(T);
  if (smem > CAP) {  // wide image: segments of the tile row, the largest multiple of 8 tiles that fits
    twb = 0;
    for (int t = 8; t < d.tw; t += 8) {
      const int w_t = 2 * d.s_w * (t - 1) + cols1;
      if ((size_t)CB * ((size_t)rows * w_t + 1) * sizeof(T) <= CAP) twb = t;
    }
    if (twb == 0) return DWM_OK;
    ws = 2 * d.s_w * (twb - 1) + cols1;
    smem = (size_t)CB * ((size_t)rows * ws + 1) * sizeof(T);
  }
  const bool wide = twb != d.tw;
  // whole rows: stage trows tile rows per CTA when they fit (the rows
  // neighbouring tile rows share are loaded once, less CTA setup per tile)
  int trows = 1;
  if (!wide && d.num_freqs <= IT_TROWS_MAX_FREQS) {
    const int rows_t = rows + (DWM_IT_TROWS - 1) * 2 * d.s_h;
    const size_t smem_t = (size_t)CB * ((size_t)rows_t * ws + 1) * sizeof(T);
    if (DWM_IT_TROWS > 1 && smem_t <= CAP) {
      trows = DWM_IT_TROWS;
      rows = rows_t;
      smem = smem_t;
    }
  }
  const int nxb = (d.tw + twb - 1) / twb;
  const int nty = (d.th + trows - 1) / trows;
  constexpr int VEC = 16 / sizeof(T);
  const int npad = d.pad_left + d.pad_right;
  const ItDivs dv{make_fastdiv((uint32_t)max(1, rows * (d.w / VEC))), make_fastdiv((uint32_t)max(1, d.w / VEC)),
                  make_fastdiv((uint32_t)max(1, rows * npad)), make_fastdiv((uint32_t)max(1, npad)),
                  make_fastdiv((uint32_t)nty)};
  // grid.y = images x CTAs per image must stay <= 65535: launch batch slices
  const int per_img = nty * nxb;
  if (per_img > 65535) return DWM_OK;  // (never at BASELINE sizes) the 1-D-grid kernel takes it
  const int imgs_per_launch = 65535 / per_img;
  const bool stream = d.num_freqs > IT_STREAM_MIN_FREQS;
  auto kern = wide ? (stream ? input_transform_smem_kernel<T, true, true, CB> : input_transform_smem_kernel<T, true, false, CB>)
                   : (stream ? input_transform_smem_kernel<T, false, true, CB> : input_transform_smem_kernel<T, false, false, CB>);
  // + the gather offset tables (non-streaming variants)
  if (!stream) smem = it_tab_offset<T>(CB, rows * ws + 1) + it_tab_bytes(d, twb, trows);
  if (int st = ensure_dynamic_smem((const void*)kern, smem)) return st;
  // warps: a divisor of the tile-step count in [4, 8] so every warp gets the
  // same number of tiles (a warp step covers 32 / CB tiles)
  const int steps = (twb + 32 / CB - 1) / (32 / CB);
  int warps = 8;
  if (steps <= 8) warps = steps < 1 ? 1 : steps;
  else
    for (int cand = 8; cand >= 4; --cand)
      if (steps % cand == 0) { warps = cand; break; }
  for (int n0 = 0; n0 < d.n; n0 += imgs_per_launch) {
    const int nb = min(imgs_per_launch, d.n - n0);
    const dim3 grid((unsigned)((d.c + CB - 1) / CB), (unsigned)(nb * per_img));
    kern<<<grid, 32 * warps, smem, s>>>(d, (const T*)x, (T*)V, rows, twb, ws, trows, n0, xmax, dv);
    DWM_CUDA_TRY(cudaGetLastError());
  }
  *used = true;
  return DWM_OK;
}

int launch_input_transform(const dwm_desc_t& d, int dtype, const void* x, void* V, cudaStream_t s,
                           uint32_t* xmax) {
  bool used = false;
  if (dtype == DWM_F64) xmax = nullptr;
  if (xmax) DWM_CUDA_TRY(cudaMemsetAsync(xmax, 0, xmax_bytes(d), s));
  // 16-channel CTAs: DWM_IT_CB=16 (experiments) or the rule below
  static const int env_cb = [] {
    const char* e = getenv("DWM_IT_CB");
    return e ? atoi(e) : 0;
  }();
  const bool cb16 = env_cb ? env_cb == 16 : it_prefers_cb16(d);
  const int st = dtype == DWM_F64 ? launch_input_smem_cb<double, 32>(d, x, V, s, &used, nullptr)
               : cb16             ? launch_input_smem_cb<float, 16>(d, x, V, s, &used, xmax)
                                  : launch_input_smem_cb<float, 32>(d, x, V, s, &used, xmax);
  if (st || used) return st;
  const int64_t n = d.tiles * d.c;
  if (dtype == DWM_F64)
    input_transform_kernel<double><<<grid_for(n, 256), 256, 0, s>>>(d, (const double*)x, (double*)V, nullptr);
  else
    input_transform_kernel<float><<<grid_for(n, 256), 256, 0, s>>>(d, (const float*)x, (float*)V, xmax);
  DWM_CUDA_TRY(cudaGetLastError());
  return DWM_OK;
}

}  // namespace dwm

namespace dwm {

// ---------------------------------------------------------------------------
// Weight gradient: the GEMM
//   gw[f][j] = sum_p dY[f][p] * X[j][p],  j = (c, ky, kx),  p = (n, oy, ox),
// X gathered on the fly from x (implicit im2col; padding by predicate).
// 64x64 output tile per CTA, 256 threads x (4 filters x 4 taps), K chunks of
// 16 positions through smem.  Each output is one FMA chain in ascending p, so
// results are deterministic and independent of the launch configuration.
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(256) weight_grad_kernel(const dwm_desc_t d, const T* __restrict__ x,
                                                          const T* __restrict__ dy, T* __restrict__ gw,
                                                          int64_t seg_len, int32_t* __restrict__ flag) {
  constexpr int BM = 64, BN = 64, BK = 16;
  __shared__ __align__(16) T As[BK][BM];
  __shared__ __align__(16) T Bs[BK][BN];
  __shared__ int p_img[BK], p_oy[BK], p_ox[BK];
  const int tid = threadIdx.x;
  const int taps = d.r_h * d.r_w;
  const int ncols = d.c * taps;
  const int f0 = blockIdx.y * BM, j0 = blockIdx.x * BN;
  const int64_t per_img = (int64_t)d.oh * d.ow;
  // K segment blockIdx.z (split-K; partial sums go to gw + z * F * ncols)
  const int64_t k_begin = (int64_t)blockIdx.z * seg_len;
  const int64_t K = min((int64_t)d.n * per_img, k_begin + seg_len);
  gw += (int64_t)blockIdx.z * d.f * ncols;

  // this thread's fixed X column (tap) for the gather: j = j0 + tid % 64
  const int jl = tid % BN;
  const int jg = j0 + jl;
  const bool j_ok = jg < ncols;
  const int jc = j_ok ? jg / taps : 0;
  const int jky = j_ok ? (jg % taps) / d.r_w : 0;
  const int jkx = j_ok ? jg % d.r_w : 0;
  const int kk = tid / BN;  // rows kk, kk+4, kk+8, kk+12 of the K chunk

  // dY loads: k fastest (coalesced along ox), filters tid/16 + 16 i
  const int ak = tid % BK;
  const int af = tid / BK;

  const int ty = tid / 16, tx = tid % 16;
  // blocked summation (like a BLAS kernel): 16-position chunk sums -> 1024-
  // position block sums -> total; error grows with ~K/1024 + 64 + 16 terms
  // instead of K for one long chain
  T acc[4][4], mid[4][4], tot[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) mid[a][b] = tot[a][b] = T(0);
  int chunk = 0;

  for (int64_t k0 = k_begin; k0 < K; k0 += BK) {
    if (tid < BK) {
      const int64_t p = k0 + tid;
      if (p < K) {
        p_img[tid] = (int)(p / per_img);
        const int rem = (int)(p % per_img);
        p_oy[tid] = rem / d.ow;
        p_ox[tid] = rem % d.ow;
      } else {
        p_img[tid] = -1;
      }
    }
    __syncthreads();
    {
      const int n = p_img[ak];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int f = f0 + af + 16 * i;
        T v = T(0);
        if (n >= 0 && f < d.f) v = dy[(((int64_t)n * d.f + f) * d.oh + p_oy[ak]) * d.ow + p_ox[ak]];
        As[ak][af + 16 * i] = v;
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int k = kk + 4 * i;
        const int nn = p_img[k];
        T v = T(0);
        if (nn >= 0 && j_ok) {
          const int row = d.s_h * p_oy[k] + jky - d.pad_top;
          const int col = d.s_w * p_ox[k] + jkx - d.pad_left;
          if (row >= 0 && row < d.h && col >= 0 && col < d.w)
            v = x[(((int64_t)nn * d.c + jc) * d.h + row) * d.w + col];
        }
        Bs[k][jl] = v;
      }
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) acc[u][v] = T(0);
#pragma unroll
    for (int k = 0; k < BK; ++k) {
      T a[4], b[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        a[q] = As[k][ty * 4 + q];
        b[q] = Bs[k][tx * 4 + q];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = fma_rn(a[u], b[v], acc[u][v]);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) mid[u][v] = add_rn(mid[u][v], acc[u][v]);
    if (++chunk == 64) {
      chunk = 0;
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          tot[u][v] = add_rn(tot[u][v], mid[u][v]);
          mid[u][v] = T(0);
        }
    }
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int f = f0 + ty * 4 + u;
    if (f >= d.f) continue;
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int j = j0 + tx * 4 + v;
      if (j < ncols) {
        const T g = add_rn(tot[u][v], mid[u][v]);
        gw[(int64_t)f * ncols + j] = g;
        if (flag && !isfinite(g)) *flag = 1;  // (only the unsplit launch passes a flag)
      }
    }
  }
}

// Fixed-order sum of the split-K partials (segment 0 first).
template <typename T>
__global__ void weight_grad_reduce_kernel(const T* __restrict__ part, T* __restrict__ gw, int64_t count,
                                          int splits, int32_t* __restrict__ flag) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  T v = part[i];
  for (int z = 1; z < splits; ++z) v = add_rn(v, part[(int64_t)z * count + i]);
  gw[i] = v;
  if (flag && !isfinite(v)) *flag = 1;
}

// Split count from the geometry only (never from the device), so a given
// problem always sums in the same order: enough CTAs for ~2 waves of 148 SMs,
// segments of at least 4096 positions.
int weight_grad_splits(const dwm_desc_t& d) {
  const int64_t ncols = (int64_t)d.c * d.r_h * d.r_w;
  const int64_t tiles = ((ncols + 63) / 64) * ((d.f + 63) / 64);
  const int64_t K = (int64_t)d.n * d.oh * d.ow;
  int64_t sp = (2 * 148 + tiles - 1) / tiles;
  sp = std::min<int64_t>(sp, (K + 4095) / 4096);
  return (int)std::max<int64_t>(1, std::min<int64_t>(sp, 256));
}

int launch_weight_grad(const dwm_desc_t& d, int dtype, const void* x, const void* dy, void* gw, void* ws,
                       size_t ws_bytes, int32_t* flag, cudaStream_t s) {
  const int ncols = d.c * d.r_h * d.r_w;
  const int splits = weight_grad_splits(d);
  const int64_t K = (int64_t)d.n * d.oh * d.ow;
  const int64_t seg = ((K + splits - 1) / splits + 15) / 16 * 16;
  const int64_t count = (int64_t)d.f * ncols;
  const size_t es = dtype == DWM_F64 ? 8 : 4;
  if (splits > 1 && (!ws || ws_bytes < (size_t)splits * count * es))
    return fail(DWM_EINVAL_SHAPE, "weight-gradient workspace too small: %zu bytes given, %zu needed", ws_bytes,
                (size_t)splits * count * es);
  const dim3 grid((unsigned)((ncols + 63) / 64), (unsigned)((d.f + 63) / 64), (unsigned)splits);
  void* dst = splits > 1 ? ws : gw;
  const unsigned rg = (unsigned)((count + 255) / 256);
  if (dtype == DWM_F64) {
    weight_grad_kernel<double><<<grid, 256, 0, s>>>(d, (const double*)x, (const double*)dy, (double*)dst, seg,
                                                     splits > 1 ? nullptr : flag);
    if (splits > 1)
      weight_grad_reduce_kernel<double><<<rg, 256, 0, s>>>((const double*)ws, (double*)gw, count, splits, flag);
  } else {
    weight_grad_kernel<float><<<grid, 256, 0, s>>>(d, (const float*)x, (const float*)dy, (float*)dst, seg,
                                                   splits > 1 ? nullptr : flag);
    if (splits > 1)
      weight_grad_reduce_kernel<float><<<rg, 256, 0, s>>>((const float*)ws, (float*)gw, count, splits, flag);
  }
  DWM_CUDA_TRY(cudaGetLastError());
  return DWM_OK;
}

}  // namespace dwm
