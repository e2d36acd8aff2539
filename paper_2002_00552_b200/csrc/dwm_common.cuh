// dwm_common.cuh -- shared device helpers for the DWM sm_100a kernels.
//
// Transform constants F(2,1), F(2,2), F(2,3) (reference transforms.py:129-208
// with nodes 0, 1, -1, infinity; r == 1 identity, transforms.py:163-167).
// All entries are 0, +-1 or +-1/2, exactly representable; applied as
// sequential FMA chains in ascending tap order, which reproduces the
// reference's BLAS small-K contraction bit for bit.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/dwm_b200.h"

namespace dwm {

// [count][row][col]; count index 1..3, unused slots zero.
// Bt: alpha x alpha, G: alpha x count, At: 2 x alpha.
static __constant__ float c_bt[4][4][4] = {
    {},
    {{1, 0}, {0, 1}},
    {{1, -1, 0}, {0, 1, 0}, {0, 1, -1}},
    {{1, 0, -1, 0}, {0, 1, 1, 0}, {0, -1, 1, 0}, {0, 1, 0, -1}},
};
static __constant__ float c_g[4][4][3] = {
    {},
    {{1}, {1}},
    {{1, 0}, {1, 1}, {0, 1}},
    {{1, 0, 0}, {0.5f, 0.5f, 0.5f}, {0.5f, -0.5f, 0.5f}, {0, 0, 1}},
};
static __constant__ float c_at[4][2][4] = {
    {},
    {{1, 0}, {0, 1}},
    {{1, 1, 0}, {0, 1, -1}},
    {{1, 1, 1, 0}, {0, 1, -1, -1}},
};

__device__ __forceinline__ float fma_rn(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ double fma_rn(double a, double b, double c) { return __fma_rn(a, b, c); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }

// Frequency offset of part p (plan order = row part major, col part minor).
__host__ __device__ __forceinline__ int part_freq_offset(const dwm_desc_t& d, int p) {
  int off = 0;
  for (int q = 0; q < p; ++q) {
    const int rp = q / d.n_col_parts, cp = q % d.n_col_parts;
    off += (d.row_parts[rp].count + 1) * (d.col_parts[cp].count + 1);
  }
  return off;
}

#define DWM_CUDA_TRY(expr)                                                  \
  do {                                                                      \
    cudaError_t _e = (expr);                                                \
    if (_e != cudaSuccess) return ::dwm::cuda_fail(_e, #expr, __FILE__, __LINE__); \
  } while (0)

int cuda_fail(cudaError_t e, const char* what, const char* file, int line);
int fail(int status, const char* fmt, ...);

// Host-side launch facts cached per (kernel, device) instead of queried on
// every launch (dwm_capi.cu): SM count, the dynamic-smem attribute (set only
// when a kernel needs more than it was last given) and CTAs per SM.
int device_sm_count(int* sms);
int ensure_dynamic_smem(const void* kernel, size_t smem);
int cached_occupancy(const void* kernel, int threads, size_t smem, int* per_sm);

// ---- packed f32x2 (FFMA2 / FADD2 / FMUL2: two lanes of work per issue slot) ----
typedef unsigned long long f2;
__device__ __forceinline__ f2 pk(float a, float b) {
  f2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float2 upk(f2 v) {
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
  return r;
}
__device__ __forceinline__ f2 fma2(f2 a, f2 b, f2 c) {
  f2 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ f2 mul2(f2 a, f2 b) {
  f2 r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f2 add2(f2 a, f2 b) {
  f2 r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f2 sub2(f2 a, f2 b) {
  f2 r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}

}  // namespace dwm
