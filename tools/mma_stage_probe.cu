// mma_stage_probe.cu -- cost of the per-stage control around the tcgen05 MMAs
// of the GEMM (dwm_gemm_tc.cu): 8 x (N=128 + N=64) kind::tf32 TS MMAs per
// 64-channel stage, then optionally a fence, a commit, and a commit/wait
// handshake with a second warp (the converter/epilogue feedback loop with no
// work).  148 CTAs x 128 threads, B resident in smem, A/D in TMEM.
//
//   ./mma_stage_probe     prints cycles per stage for each mode
#include <cstdio>

#include "../paper_2002_00552_b200/csrc/dwm_sm100.cuh"

using namespace dwm::sm100;

// mode bits: 1 fence per stage, 2 commit per stage, 4 handshake (MMA waits a
// barrier the helper warp arrives on after observing the commit of stage-2),
// 8 N=128 only (no N=64 MMA), 16 fresh accumulator per stage in 2 buffers,
// 32 three smem B stages (descriptor changes per stage)
__global__ void k(int iters, int mode, long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t done[3], ready[2];
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid / 32;
  for (int e = tid; e < 3 * 2 * 128 * 32; e += blockDim.x) ((float*)smem)[e] = 1.0f / (1 + (e % 7));
  if (tid == 0) {
    for (int i = 0; i < 3; ++i) mbar_init(&done[i], 1);
    for (int i = 0; i < 2; ++i) mbar_init(&ready[i], 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(&tmem_base);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t t = tmem_base;
  const uint32_t i128 = idesc_tf32(128, 128), i64 = idesc_tf32(128, 64);
  long long t0 = clock64();
  if (warp == 0) {
    for (int it = 0; it < iters; ++it) {
      if ((mode & 4) && it >= 2) mbar_wait(&ready[it % 2], ((it - 2) / 2) & 1);
      if (mode & 1) tc_fence_after();
      const int sb = (mode & 32) ? it % 3 : 0;
      const uint32_t dacc = t + ((mode & 16) ? 128 * (it & 1) : 0);
      if (elect_one()) {
        for (int h = 0; h < 2; ++h) {
          const uint64_t du = sdesc_sw128(smem_u32(smem + (sb * 2 + h) * 16384));
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const bool fresh = (mode & 16) && h == 0 && kk == 0;
            mma_tf32_ts(dacc, t + 256 + 32 * h + 8 * kk, du + 2 * kk, i128, fresh ? 0u : 1u);
            if (!(mode & 8)) mma_tf32_ts(dacc + 64, t + 320 + 32 * h + 8 * kk, du + 2 * kk, i64, 1u);
          }
        }
        if (mode & 2) mma_commit(&done[it % 3]);
      }
      __syncwarp();
    }
    if (elect_one()) mma_commit(&done[iters % 3]);
    __syncwarp();
  } else if (warp == 1 && (mode & 4)) {
    // helper: stage it done -> ready for stage it + 2
    for (int it = 0; it < iters; ++it) {
      mbar_wait(&done[it % 3], (it / 3) & 1);
      if (tid % 32 == 0) mbar_arrive(&ready[it % 2]);
      __syncwarp();
    }
  }
  __syncthreads();
  if (warp == 0) {
    // wait for everything: the final commit (its own phase of done[iters % 3])
    mbar_wait(&done[iters % 3], (mode & 2) ? ((iters / 3) & 1) : 0);
  }
  __syncthreads();
  if (tid == 0) cyc[blockIdx.x] = clock64() - t0;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(t);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* cyc;
  cudaMalloc(&cyc, sizeof(long long) * sms);
  const int smem = 1024 + 3 * 2 * 16384;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int modes[] = {0, 8, 1, 2, 3, 16, 32, 2 | 4, 1 | 2 | 4, 1 | 2 | 4 | 16, 1 | 2 | 4 | 16 | 32, 1 | 2 | 4 | 8 | 16 | 32};
  for (int mode : modes) {
    const int iters = 4000;
    k<<<sms, 128, smem>>>(10, mode, cyc);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<<<sms, 128, smem>>>(iters, mode, cyc);
    cudaEventRecord(e1);
    if (cudaEventSynchronize(e1) != cudaSuccess) {
      printf("mode %d: error %s\n", mode, cudaGetErrorString(cudaGetLastError()));
      return 1;
    }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    long long c0;
    cudaMemcpy(&c0, cyc, sizeof(c0), cudaMemcpyDeviceToHost);
    const double flops = 2.0 * 128 * 8 * (mode & 8 ? 128 : 192) * 8.0 * iters * sms;
    printf("mode %2d (%s%s%s%s%s%s): %6.1f cycles/stage (SM clock), %7.1f TFLOP/s\n", mode, mode & 1 ? "fence " : "",
           mode & 2 ? "commit " : "", mode & 4 ? "handshake " : "", mode & 8 ? "N128-only " : "",
           mode & 16 ? "fresh-acc " : "", mode & 32 ? "3-stage-B" : "", (double)c0 / iters, flops / ms / 1e9);
  }
  return 0;
}
