// ring_probe.cu -- MMA -> epilogue accumulator ring: how deep must it be?
// MMA warp: per chunk, 12 tcgen05.mma (M=128,N=64,K=8, TS) into acc[c % R], commit acc_full;
// 8 epilogue warps: wait acc_full, tcgen05.ld their 32 columns, arrive acc_empty.
#include <cstdio>
#include "../paper_2002_00552_b200/csrc/dwm_sm100.cuh"
using namespace dwm::sm100;

__device__ __forceinline__ void ld32(uint32_t a, float (&v)[32]) {
  uint32_t r[32];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
    : "=r"(r[0]),"=r"(r[1]),"=r"(r[2]),"=r"(r[3]),"=r"(r[4]),"=r"(r[5]),"=r"(r[6]),"=r"(r[7]),"=r"(r[8]),"=r"(r[9]),"=r"(r[10]),"=r"(r[11]),"=r"(r[12]),"=r"(r[13]),"=r"(r[14]),"=r"(r[15]),
      "=r"(r[16]),"=r"(r[17]),"=r"(r[18]),"=r"(r[19]),"=r"(r[20]),"=r"(r[21]),"=r"(r[22]),"=r"(r[23]),"=r"(r[24]),"=r"(r[25]),"=r"(r[26]),"=r"(r[27]),"=r"(r[28]),"=r"(r[29]),"=r"(r[30]),"=r"(r[31]) : "r"(a));
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

template <int R, int MODE>
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
      if (MODE == 0) {
        float v[16], w[16];
        tmem_ld16(la + 64 * slot, v);
        tmem_ld16(la + 64 * slot + 16, w);
        tmem_ld_wait();
        for (int j = 0; j < 16; ++j) acc += v[j] + w[j];
      } else if (MODE == 1) {
        float v[32];
        ld32(la + 64 * slot, v);
        tmem_ld_wait();
        for (int j = 0; j < 32; ++j) acc += v[j];
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
    }
  }
  if (acc == 1234.f) sink[0] = acc;
  tc_fence_before(); __syncthreads();
  if (warp == 0) tmem_dealloc<512>(t);
}

template <int R, int MODE = 0>
void run(int sms, int per) {
  float* sink; cudaMalloc(&sink, 4);
  const int smem = 1024 + 64 * 128;
  const int chunks = 48000 / per;
  cudaFuncSetAttribute(k<R, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<R, MODE><<<sms, 288, smem>>>(10, per, sink);
  cudaEventRecord(e0);
  k<R, MODE><<<sms, 288, smem>>>(chunks, per, sink);
  cudaEventRecord(e1);
  if (cudaEventSynchronize(e1) != cudaSuccess) { printf("error\n"); exit(1); }
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("ring %d mode %d, %2d MMAs/chunk: %.1f cycles/MMA\n", R, MODE, per, ms * 1e-3 * 1.965e9 / ((double)chunks * per));
}

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int per : {12, 24}) { run<2, 0>(sms, per); run<2, 1>(sms, per); }
  return 0;
}
