// ring_probe.cu -- MMA -> epilogue accumulator ring: how deep must it be?
// MMA warp: per chunk, 12 tcgen05.mma (M=128,N=64,K=8, TS) into acc[c % R], commit acc_full;
// 8 epilogue warps: wait acc_full, tcgen05.ld their 32 columns, arrive acc_empty.
#include <cstdio>
#include "../paper_2002_00552_b200/csrc/dwm_sm100.cuh"
using namespace dwm::sm100;

template <int R>
__global__ void k(int chunks, int per, float* sink) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t full[R], empty[R];
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  for (int e = tid; e < 64 * 32; e += blockDim.x) ((float*)smem)[e] = 1.0f / (1 + (e % 7));
  if (tid == 0) { for (int i = 0; i < R; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 8); } fence_barrier_init(); }
  if (warp == 0) tmem_alloc<512>(&tmem_base);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t t = tmem_base;
  float acc = 0;
  if (warp == 8) {
    const uint32_t idesc = idesc_tf32(128, 64);
    const uint64_t b0 = sdesc_sw128(smem_u32(smem));
    for (int c = 0; c < chunks; ++c) {
      const int slot = c % R;
      mbar_wait(&empty[slot], ((c / R) & 1) ^ 1);
      tc_fence_after();
      if (elect_one()) {
        for (int j = 0; j < per; ++j) mma_tf32_ts(t + 64 * slot, t + 448 + 8 * (j & 3), b0 + 2 * (j & 3), idesc, j != 0);
        mma_commit(&full[slot]);
      }
      __syncwarp();
    }
  } else if (warp < 8) {
    const uint32_t la = t + ((uint32_t)(32 * (warp % 4)) << 16) + 32 * (warp / 4);
    for (int c = 0; c < chunks; ++c) {
      const int slot = c % R;
      mbar_wait(&full[slot], (c / R) & 1);
      tc_fence_after();
      float v[16], w[16];
      tmem_ld16(la + 64 * slot, v);
      tmem_ld16(la + 64 * slot + 16, w);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
      for (int j = 0; j < 16; ++j) acc += v[j] + w[j];
    }
  }
  if (acc == 1234.f) sink[0] = acc;
  tc_fence_before(); __syncthreads();
  if (warp == 0) tmem_dealloc<512>(t);
}

template <int R>
void run(int sms, int per) {
  float* sink; cudaMalloc(&sink, 4);
  const int smem = 1024 + 64 * 128;
  const int chunks = 48000 / per;
  cudaFuncSetAttribute(k<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<R><<<sms, 288, smem>>>(10, per, sink);
  cudaEventRecord(e0);
  k<R><<<sms, 288, smem>>>(chunks, per, sink);
  cudaEventRecord(e1);
  if (cudaEventSynchronize(e1) != cudaSuccess) { printf("error\n"); exit(1); }
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("ring %d, %2d MMAs/chunk: %.1f cycles/MMA\n", R, per, ms * 1e-3 * 1.965e9 / ((double)chunks * per));
}

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int per : {12, 24}) { run<1>(sms, per); run<2>(sms, per); run<3>(sms, per); run<4>(sms, per); }
  return 0;
}
