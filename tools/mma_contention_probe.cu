// mma_contention_probe.cu -- which shared resource slows the tcgen05 GEMM's
// MMA stream?  The MMA loop of dwm_gemm_tc.cu (per 64-channel stage: 8 x
// (N=128 + N=64) kind::tf32 TS MMAs, one commit) runs against helper warps
// that, paced by the stage commits like the real roles, generate one kind of
// traffic each:
//   bit 1: "converter"  4 warps, tcgen05.st of 128 lanes x 128 columns (A slot) per stage
//   bit 2: "epilogue"   8 warps, tcgen05.ld of 128 lanes x 128 columns (accumulator) per stage
//   bit 4: "smem"       4 warps, LDS.128 of 32 KB per stage (the converter's V reads)
//   bit 8: "tma"        1 warp, 64 KB of TMA-like cp.async.bulk global->smem per stage
// Prints cycles per stage for each combination.
#include <cstdio>

#include "../paper_2002_00552_b200/csrc/dwm_sm100.cuh"

using namespace dwm::sm100;

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

__global__ void __launch_bounds__(512, 1) k(int iters, int mode, const float* gsrc, long long* cyc, float* sink) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  // smem: [0, 96 KB) B operand stages (3 x 2 atoms x 16 KB), [96 KB, 192 KB) TMA landing zone
  __shared__ uint64_t done[16], tbar[2];
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  for (int e = tid; e < 96 * 1024 / 4; e += blockDim.x) ((float*)smem)[e] = 1.0f / (1 + (e % 7));
  if (tid == 0) {
    for (int i = 0; i < 16; ++i) mbar_init(&done[i], 1);
    for (int i = 0; i < 2; ++i) mbar_init(&tbar[i], 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(&tmem_base);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t t = tmem_base;
  const uint32_t i128 = idesc_tf32(128, 128), i64 = idesc_tf32(128, 64);
  const long long t0 = clock64();
  float acc = 0.f;
  if (warp == 13) {
    // MMA issuer: D buffer alternates (cols 0/128), A slots at 256/384
    for (int it = 0; it < iters; ++it) {
      const int sb = it % 3;
      const uint32_t dacc = t + 128 * (it & 1), a = t + 256 + 128 * (it & 1);
      if (elect_one()) {
        for (int h = 0; h < 2; ++h) {
          const uint64_t du = sdesc_sw128(smem_u32(smem + (sb * 2 + h) * 16384));
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            mma_tf32_ts(dacc, a + 32 * h + 8 * kk, du + 2 * kk, i128, (h == 0 && kk == 0) ? 0u : 1u);
            mma_tf32_ts(dacc + 64, a + 64 + 32 * h + 8 * kk, du + 2 * kk, i64, 1u);
          }
        }
        mma_commit(&done[it % 16]);
      }
      __syncwarp();
      // pace: at most 2 stages in flight (the real kernel's A-slot/acc ring)
      if (it >= 1) mbar_wait(&done[(it - 1) % 16], ((it - 1) / 16) & 1);
    }
    mbar_wait(&done[(iters - 1) % 16], ((iters - 1) / 16) & 1);
    // timed by the MMA warp itself (a clock read after __syncthreads is taken
    // before the deferred barrier completes)
    if (lane == 0) cyc[blockIdx.x] = clock64() - t0;
  } else if (warp < 4 && (mode & 1)) {
    // converter: after stage it completes, store the A slot of stage it + 2
    const uint32_t la = t + ((uint32_t)(32 * warp) << 16);
    float v[16];
    for (int j = 0; j < 16; ++j) v[j] = (float)(lane + j);
    for (int it = 0; it < iters; ++it) {
      mbar_wait(&done[it % 16], (it / 16) & 1);
      const uint32_t a = la + 256 + 128 * (it & 1);
#pragma unroll
      for (int c = 0; c < 128; c += 16) tmem_st16(a + c, v);
      tmem_st_wait();
    }
  } else if (warp >= 4 && warp < 12 && (mode & 2)) {
    // epilogue: drain the accumulator buffer of stage it (64 of its 128 columns per warp)
    const int quad = warp % 4, half = (warp - 4) / 4;
    const uint32_t la = t + ((uint32_t)(32 * quad) << 16);
    for (int it = 0; it < iters; ++it) {
      mbar_wait(&done[it % 16], (it / 16) & 1);
      const uint32_t d = la + 128 * (it & 1) + 64 * half;
      float v[16];
#pragma unroll
      for (int c = 0; c < 64; c += 16) {
        tmem_ld16(d + c, v);
        tmem_ld_wait();
        for (int j = 0; j < 16; ++j) acc += v[j];
      }
    }
  } else if (warp >= 4 && warp < 8 && (mode & 4)) {
    // smem readers: 32 KB of LDS.128 per stage (8 KB per warp)
    for (int it = 0; it < iters; ++it) {
      mbar_wait(&done[it % 16], (it / 16) & 1);
      const float4* p = (const float4*)(smem + ((it % 3) * 2) * 16384 + (warp - 4) * 8192);
      for (int e = lane; e < 512; e += 32) {
        const float4 q = p[e];
        acc += q.x + q.y + q.z + q.w;
      }
    }
  } else if (warp == 12 && (mode & 8)) {
    // TMA-like: 32 KB global (L2-resident) -> smem per stage (2 x 16 KB bulk copies)
    for (int it = 0; it < iters; ++it) {
      // free-running (not gated on done[]: a lagging reader would alias phases)
      if (elect_one()) {
        const int b = it & 1;
        if (it >= 2) mbar_wait(&tbar[b], ((it - 2) / 2) & 1);
        mbar_arrive_expect_tx(&tbar[b], 32768);
        for (int j = 0; j < 2; ++j)
          bulk_g2s(smem + 96 * 1024 + j * 16384 + b * 0, gsrc + ((size_t)(blockIdx.x * 64 + it % 8) * 4 + j) * 4096,
                   16384, &tbar[b]);
      }
      __syncwarp();
    }
    // drain the copies still in flight before the CTA may exit
    for (int it = iters - 2 < 0 ? 0 : iters - 2; it < iters; ++it) mbar_wait(&tbar[it & 1], (it / 2) & 1);
  }
  __syncthreads();
  if (acc == 12345.f) sink[blockIdx.x] = acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(t);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* cyc;
  float *sink, *g;
  cudaMalloc(&cyc, sizeof(long long) * sms);
  cudaMalloc(&sink, 4096);
  const size_t gbytes = (size_t)sms * 64 * 4 * 4096 * 4 + (1 << 20);
  cudaMalloc(&g, gbytes);
  cudaMemset(g, 0, gbytes);
  const int smem = 1024 + 192 * 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int modes[] = {0, 1, 2, 4, 8, 1 | 2, 1 | 4, 1 | 2 | 4, 1 | 2 | 4 | 8};
  for (int mode : modes) {
    const int iters = 3000;
    k<<<sms, 512, smem>>>(10, mode, g, cyc, sink);
    k<<<sms, 512, smem>>>(iters, mode, g, cyc, sink);
    if (cudaDeviceSynchronize() != cudaSuccess) {
      printf("mode %d: error %s\n", mode, cudaGetErrorString(cudaGetLastError()));
      return 1;
    }
    long long c0;
    cudaMemcpy(&c0, cyc, sizeof(c0), cudaMemcpyDeviceToHost);
    printf("mode %2d (%s%s%s%s): %6.1f cycles/stage\n", mode, mode & 1 ? "tmem-st " : "", mode & 2 ? "tmem-ld " : "",
           mode & 4 ? "lds " : "", mode & 8 ? "tma " : "", (double)c0 / iters);
  }
  return 0;
}
