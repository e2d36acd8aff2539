// Microbenchmark: FP32 issue throughput on sm_100a for FFMA (scalar, 3-reg),
// FFMA2 (packed f32x2), FADD and FADD2.  Reports TFLOP/s (FMA = 2 flops per lane).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long pk(float a, float b) {
  unsigned long long r; asm volatile("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b)); return r;
}

template <int MODE>
__global__ void bench(float* out, int iters, float s) {
  float a[16];
  unsigned long long p[8];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-3f + i;
#pragma unroll
  for (int i = 0; i < 8; ++i) p[i] = pk(a[2 * i], a[2 * i + 1]);
  const float b = s, c = s * 0.5f;
  const unsigned long long bb = pk(b, b), cc = pk(c, c);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (MODE == 0) {
#pragma unroll
        for (int i = 0; i < 16; ++i) a[i] = __fmaf_rn(a[i], b, c);
      } else if (MODE == 1) {
#pragma unroll
        for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(p[i]) : "l"(bb), "l"(cc));
      } else if (MODE == 2) {
#pragma unroll
        for (int i = 0; i < 16; ++i) a[i] = __fadd_rn(a[i], c);
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(p[i]) : "l"(cc));
      }
    }
  }
  float s2 = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s2 += a[i];
#pragma unroll
  for (int i = 0; i < 8; ++i) { float x, y; asm("mov.b64 {%0,%1}, %2;" : "=f"(x), "=f"(y) : "l"(p[i])); s2 += x + y; }
  if (s2 == 12345.f) out[0] = s2;
}

int main() {
  float* out; cudaMalloc(&out, 4);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 4096, threads = 512, blocks = sms * 4;
  const char* names[] = {"FFMA", "FFMA2", "FADD", "FADD2"};
  for (int mode = 0; mode < 4; ++mode) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (mode == 0) bench<0><<<blocks, threads>>>(out, iters, 0.999f);
      if (mode == 1) bench<1><<<blocks, threads>>>(out, iters, 0.999f);
      if (mode == 2) bench<2><<<blocks, threads>>>(out, iters, 0.999f);
      if (mode == 3) bench<3><<<blocks, threads>>>(out, iters, 0.999f);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
    }
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double lane_ops = (double)blocks * threads * iters * 8 * 16;  // 16 fp32 results per k
    const double flops = lane_ops * (mode == 0 || mode == 1 ? 2 : 1);
    printf("%-6s %8.3f ms  %7.2f T lane-results/s  %7.2f TFLOP/s\n", names[mode], ms, lane_ops / ms / 1e9, flops / ms / 1e9);
  }
  return 0;
}
