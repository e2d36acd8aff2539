// commit_probe.cu -- does tcgen05.commit (or the mbarrier round trip around it)
// throttle back-to-back tcgen05.mma issue?  TS mode, M=128, N=64, K=8.
#include <cstdio>
#include "../paper_2002_00552_b200/csrc/dwm_sm100.cuh"
using namespace dwm::sm100;

// mode 0: no commits; 1: commit to a dummy barrier every `per` MMAs;
// 2: commit every `per` MMAs and wait for that commit before issuing more (full drain)
// 3: like 1, but alternate 2 accumulators (ring) and wait for the commit of the previous use of a slot
__global__ void k(int iters, int per, int mode, float* sink) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar[3];
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid / 32;
  for (int e = tid; e < 64 * 32; e += blockDim.x) ((float*)smem)[e] = 1.0f / (1 + (e % 7));
  if (tid == 0) { mbar_init(&bar[0], 1); mbar_init(&bar[1], 1); mbar_init(&bar[2], 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc<512>(&tmem_base);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t t = tmem_base;
  if (warp == 0) {
    if (tid == 0) {
      const uint32_t idesc = idesc_tf32(128, 64);
      const uint32_t b = smem_u32(smem);
      uint32_t n = 0, ph[2] = {0, 0};
      for (int it = 0; it < iters; ++it) {
        uint32_t dcol = 0;
        if (mode == 3 || mode == 5) dcol = 64 * (it & 1);
        if (mode == 6) dcol = 64 * (it & 3);
        const bool reset_ok = mode != 4;
        for (int j = 0; j < per; ++j)
          mma_tf32_ts(t + dcol, t + 256 + 8 * (j & 3), sdesc_sw128(b + 32 * (j & 3)), idesc, reset_ok ? (j != 0) : 1);
        if (mode >= 1 && mode <= 3) {
          const int slot = mode == 3 ? (it & 1) : 0;
          mma_commit(&bar[slot]);
          if (mode == 2) { mbar_wait(&bar[0], ph[0]); ph[0] ^= 1; }
          if (mode == 3 && it >= 1) { const int o = (it - 1) & 1; mbar_wait(&bar[o], ph[o]); ph[o] ^= 1; }
        }
        ++n;
      }
      mma_commit(&bar[2]);
    }
    __syncwarp();
  }
  mbar_wait(&bar[2], 0);
  tc_fence_after();
  if (warp == 0) { float v[16]; tmem_ld16(t, v); tmem_ld_wait(); if (tid == 0) sink[blockIdx.x] = v[0]; }
  tc_fence_before(); __syncthreads();
  if (warp == 0) tmem_dealloc<512>(t);
}

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(pred));
  return pred != 0;
}

// warp-converged issue loop: every lane computes the (uniform) operands, one elected lane issues
__global__ void kw(int iters, int per, float* sink) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar[3];
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid / 32;
  for (int e = tid; e < 64 * 32; e += blockDim.x) ((float*)smem)[e] = 1.0f / (1 + (e % 7));
  if (tid == 0) { mbar_init(&bar[0], 1); mbar_init(&bar[1], 1); mbar_init(&bar[2], 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc<512>(&tmem_base);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t t = tmem_base;
  if (warp == 0) {
    const uint32_t idesc = idesc_tf32(128, 64);
    const uint64_t b0 = sdesc_sw128(smem_u32(smem));
    for (int it = 0; it < iters; ++it) {
      const uint32_t dcol = 64 * (it & 1);
      for (int j = 0; j < per; ++j) {
        if (elect_one()) mma_tf32_ts(t + dcol, t + 256 + 8 * (j & 3), b0 + 2 * (j & 3), idesc, j != 0);
        __syncwarp();
      }
      if (elect_one()) mma_commit(&bar[it & 1]);
      __syncwarp();
    }
    if (elect_one()) mma_commit(&bar[2]);
    __syncwarp();
  }
  mbar_wait(&bar[2], 0);
  tc_fence_after();
  if (warp == 0) { float v[16]; tmem_ld16(t, v); tmem_ld_wait(); if (tid == 0) sink[blockIdx.x] = v[0]; }
  tc_fence_before(); __syncthreads();
  if (warp == 0) tmem_dealloc<512>(t);
}

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* sink; cudaMalloc(&sink, 4 * 1024);
  const int smem = 1024 + 64 * 128;
  const char* names[] = {"no commit", "commit", "commit+drain", "commit ring-2", "never reset", "reset ring-2", "reset ring-4"};
  for (int mode = 0; mode < 7; ++mode)
    for (int per : {4, 6, 12, 24}) {
      const int total = 48000, iters = total / per;
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      k<<<sms, 128, smem>>>(10, per, mode, sink);
      cudaEventRecord(e0);
      k<<<sms, 128, smem>>>(iters, per, mode, sink);
      cudaEventRecord(e1);
      if (cudaEventSynchronize(e1) != cudaSuccess) { printf("error\n"); return 1; }
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      const double flops = 2.0 * 128 * 64 * 8 * (double)iters * per * sms;
      printf("%-14s per=%2d: %7.1f TFLOP/s  (%.1f cycles/MMA)\n", names[mode], per, flops / ms / 1e9,
             ms * 1e-3 * 1.965e9 / ((double)iters * per));
    }
  for (int per : {4, 6, 12, 24}) {
    const int total = 48000, iters = total / per;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    kw<<<sms, 128, smem>>>(10, per, sink);
    cudaEventRecord(e0);
    kw<<<sms, 128, smem>>>(iters, per, sink);
    cudaEventRecord(e1);
    if (cudaEventSynchronize(e1) != cudaSuccess) { printf("error\n"); return 1; }
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * 128 * 64 * 8 * (double)iters * per * sms;
    printf("warp-elect     per=%2d: %7.1f TFLOP/s  (%.1f cycles/MMA)\n", per, flops / ms / 1e9,
           ms * 1e-3 * 1.965e9 / ((double)iters * per));
  }
  return 0;
}
