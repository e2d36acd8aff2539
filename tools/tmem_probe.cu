// tmem_probe.cu -- TMEM load/store bandwidth per SM on B200 for tcgen05.ld/st
// 32x32b shapes x16/x32/x64 with one wait per batch of `cols` columns.
#include <cstdio>
#include "../paper_2002_00552_b200/csrc/dwm_sm100.cuh"
using namespace dwm::sm100;

template <int X>
__device__ __forceinline__ void ld_x(uint32_t a, uint32_t (&r)[X]);
template <>
__device__ __forceinline__ void ld_x<32>(uint32_t a, uint32_t (&r)[32]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
    : "=r"(r[0]),"=r"(r[1]),"=r"(r[2]),"=r"(r[3]),"=r"(r[4]),"=r"(r[5]),"=r"(r[6]),"=r"(r[7]),"=r"(r[8]),"=r"(r[9]),"=r"(r[10]),"=r"(r[11]),"=r"(r[12]),"=r"(r[13]),"=r"(r[14]),"=r"(r[15]),
      "=r"(r[16]),"=r"(r[17]),"=r"(r[18]),"=r"(r[19]),"=r"(r[20]),"=r"(r[21]),"=r"(r[22]),"=r"(r[23]),"=r"(r[24]),"=r"(r[25]),"=r"(r[26]),"=r"(r[27]),"=r"(r[28]),"=r"(r[29]),"=r"(r[30]),"=r"(r[31]) : "r"(a));
}

// each warp: `iters` x (load 64 columns of its 32 lanes as 2 x32 loads, one wait), optional store back
__global__ void bw(int iters, int mode, float* sink) {
  __shared__ uint32_t base;
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc<512>(&base);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t a = base + ((uint32_t)(32 * (warp % 4)) << 16) + 128 * ((warp / 4) % 4);
  uint32_t acc = 0;
  for (int it = 0; it < iters; ++it) {
    uint32_t r0[32], r1[32];
    ld_x<32>(a, r0);
    ld_x<32>(a + 32, r1);
    tmem_ld_wait();
#pragma unroll
    for (int j = 0; j < 32; ++j) acc += r0[j] ^ r1[j];
    if (mode == 1) {
      float v[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(r0[j] + 1);
      tmem_st16(a, v); tmem_st16(a + 16, v); tmem_st16(a + 32, v); tmem_st16(a + 48, v);
      tmem_st_wait();
    }
  }
  if (acc == 12345u) sink[0] = 1.f;
  tc_fence_before(); __syncthreads();
  if (warp == 0) tmem_dealloc<512>(base);
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* sink; cudaMalloc(&sink, 4);
  for (int mode = 0; mode < 2; ++mode)
    for (int warps : {4, 8, 16}) {
      const int iters = 20000;
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      bw<<<sms, 32 * warps>>>(10, mode, sink);
      cudaEventRecord(e0);
      bw<<<sms, 32 * warps>>>(iters, mode, sink);
      cudaEventRecord(e1);
      if (cudaEventSynchronize(e1) != cudaSuccess) { printf("error\n"); return 1; }
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      const double bytes = (double)warps * 32 * 64 * 4 * iters * (mode ? 2 : 1);
      printf("%s x32 loads, %2d warps/SM: %.1f B/cycle/SM\n", mode ? "ld+st" : "ld   ", warps, bytes / (ms * 1e-3 * 1.965e9));
    }
  return 0;
}
