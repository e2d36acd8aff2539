// tc_probe.cu -- validate the tcgen05 kind::tf32 building blocks in
// paper_2002_00552_b200/csrc/dwm_sm100.cuh on the B200 and measure the
// TF32 tensor-pipe throughput (the roofline peak for the 3xTF32 GEMM).
//
//   ./tc_probe            correctness (M=128, N in {64,128,256}, K=32) +
//                         fp32->tf32 input rounding probe + throughput sweep
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <string>
#include <vector>

#include "../paper_2002_00552_b200/csrc/dwm_sm100.cuh"

using namespace dwm::sm100;

// One CTA, 128 threads.  A: [128][32] fp32, B: [N][32] fp32 (row-major, K
// contiguous) staged into SW128 smem; D = A * B^T (K = 32, four MMAs) -> out [128][N].
template <int N>
__global__ void gemm_once(const float* A, const float* B, float* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  float* sA = (float*)smem;
  float* sB = (float*)(smem + 128 * 128);
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid / 32;
  for (int e = tid; e < 128 * 32; e += blockDim.x) {
    int r = e / 32, k = e % 32;
    *(float*)((uint8_t*)sA + sw128_offset(r, k)) = A[e];
  }
  for (int e = tid; e < N * 32; e += blockDim.x) {
    int r = e / 32, k = e % 32;
    *(float*)((uint8_t*)sB + sw128_offset(r, k)) = B[e];
  }
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<256>(&tmem_base);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic smem writes -> async proxy
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tmem_base;
  if (tid == 0) {
    const uint32_t idesc = idesc_tf32(128, N);
    for (int k = 0; k < 4; ++k) {
      mma_tf32(tbase, sdesc_sw128(smem_u32(sA) + 32 * k), sdesc_sw128(smem_u32(sB) + 32 * k), idesc, k > 0);
    }
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  // warp w reads lanes 32w..32w+31
  for (int c0 = 0; c0 < N; c0 += 16) {
    float v[16];
    tmem_ld16(tbase + ((uint32_t)(32 * warp) << 16) + c0, v);
    tmem_ld_wait();
    for (int j = 0; j < 16; ++j) out[(32 * warp + (tid % 32)) * N + c0 + j] = v[j];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<256>(tbase);
}

// Throughput: every CTA issues `iters` x 4 MMAs (M=128, N, K=8 each) on resident smem.
template <int N>
__global__ void mma_rate(int iters, float* sink) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid / 32;
  for (int e = tid; e < (128 + N) * 32; e += blockDim.x) ((float*)smem)[e] = 1.0f / (1 + (e % 7));
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<256>(&tmem_base);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tmem_base;
  if (warp == 0) {
    if (tid == 0) {
      const uint32_t idesc = idesc_tf32(128, N);
      const uint32_t a = smem_u32(smem), b = smem_u32(smem + 128 * 128);
      for (int it = 0; it < iters; ++it)
        for (int k = 0; k < 4; ++k) mma_tf32(tbase, sdesc_sw128(a + 32 * k), sdesc_sw128(b + 32 * k), idesc, 1);
      mma_commit(&bar);
    }
    __syncwarp();
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  if (warp == 0) {  // tcgen05.ld is .sync.aligned: the whole warp executes it
    float v[16];
    tmem_ld16(tbase, v);
    tmem_ld_wait();
    if (tid == 0) sink[blockIdx.x] = v[0];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<256>(tbase);
}

// TS mode: A [128][32] written to TMEM columns [256, 288) by tcgen05.st (thread m -> lane m),
// B [N][32] in SW128 smem; D = A * B^T into TMEM columns [0, N).
template <int N>
__global__ void gemm_once_ts(const float* A, const float* B, float* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  float* sB = (float*)smem;
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid / 32;
  for (int e = tid; e < N * 32; e += blockDim.x) {
    int r = e / 32, k = e % 32;
    *(float*)((uint8_t*)sB + sw128_offset(r, k)) = B[e];
  }
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(&tmem_base);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tmem_base;
  const uint32_t lane_addr = tbase + ((uint32_t)(32 * warp) << 16);
  for (int c0 = 0; c0 < 32; c0 += 16) {
    float v[16];
    for (int j = 0; j < 16; ++j) v[j] = A[tid * 32 + c0 + j];
    tmem_st16(lane_addr + 256 + c0, v);
  }
  tmem_st_wait();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) {
    if (tid == 0) {
      const uint32_t idesc = idesc_tf32(128, N);
      for (int k = 0; k < 4; ++k) mma_tf32_ts(tbase, tbase + 256 + 8 * k, sdesc_sw128(smem_u32(sB) + 32 * k), idesc, k > 0);
      mma_commit(&bar);
    }
    __syncwarp();
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  for (int c0 = 0; c0 < N; c0 += 16) {
    float v[16];
    tmem_ld16(lane_addr + c0, v);
    tmem_ld_wait();
    for (int j = 0; j < 16; ++j) out[tid * N + c0 + j] = v[j];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tbase);
}

template <int N>
__global__ void mma_rate_ts(int iters, float* sink) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid / 32;
  for (int e = tid; e < N * 32; e += blockDim.x) ((float*)smem)[e] = 1.0f / (1 + (e % 7));
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(&tmem_base);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tmem_base;
  if (warp == 0) {
    if (tid == 0) {
      const uint32_t idesc = idesc_tf32(128, N);
      const uint32_t b = smem_u32(smem);
      for (int it = 0; it < iters; ++it)
        for (int k = 0; k < 4; ++k) mma_tf32_ts(tbase, tbase + 256 + 8 * k, sdesc_sw128(b + 32 * k), idesc, 1);
      mma_commit(&bar);
    }
    __syncwarp();
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  if (warp == 0) {
    float v[16];
    tmem_ld16(tbase, v);
    tmem_ld_wait();
    if (tid == 0) sink[blockIdx.x] = v[0];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tbase);
}

// TMEM bandwidth: each warp repeatedly loads (and optionally stores back) 64 columns of its lanes.
__global__ void tmem_bw(int iters, int do_store, float* sink) {
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid / 32;
  if (warp == 0) tmem_alloc<512>(&tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t a = tmem_base + ((uint32_t)(32 * (warp % 4)) << 16) + 128 * (warp / 4);
  float acc = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 64; c += 16) {
      float v[16];
      tmem_ld16(a + c, v);
      tmem_ld_wait();
      if (do_store) {
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] += 1.0f;
        tmem_st16(a + c, v);
      } else {
#pragma unroll
        for (int j = 0; j < 16; ++j) acc += v[j];
      }
    }
  }
  if (do_store) tmem_st_wait();
  if (acc == 123.f) sink[0] = acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem_base);
}

static float tf32_round_host(float x, bool rn) {
  uint32_t u;
  memcpy(&u, &x, 4);
  if (rn) u += 0xFFF + ((u >> 13) & 1);
  u &= 0xFFFFE000u;
  float r;
  memcpy(&r, &u, 4);
  return r;
}

template <int N>
int check(bool tf32_inputs) {
  std::vector<float> A(128 * 32), B(N * 32), D(128 * N);
  srand(1 + N);
  for (auto& a : A) {
    a = (rand() % 2001 - 1000) / 997.0f;
    if (tf32_inputs) a = tf32_round_host(a, true);
  }
  for (auto& b : B) {
    b = (rand() % 2001 - 1000) / 991.0f;
    if (tf32_inputs) b = tf32_round_host(b, true);
  }
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4);
  cudaMalloc(&dB, B.size() * 4);
  cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  const int smem = 1024 + (128 + N) * 128;
  cudaFuncSetAttribute(gemm_once<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  gemm_once<N><<<1, 128, smem>>>(dA, dB, dD);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("N=%d: CUDA error %s\n", N, cudaGetErrorString(e));
    return 1;
  }
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  double maxerr_rn = 0, maxerr_tr = 0, maxerr_exact = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < N; ++n) {
      double rn = 0, tr = 0, ex = 0;
      for (int k = 0; k < 32; ++k) {
        rn += (double)tf32_round_host(A[m * 32 + k], true) * tf32_round_host(B[n * 32 + k], true);
        tr += (double)tf32_round_host(A[m * 32 + k], false) * tf32_round_host(B[n * 32 + k], false);
        ex += (double)A[m * 32 + k] * B[n * 32 + k];
      }
      maxerr_rn = fmax(maxerr_rn, fabs(D[m * N + n] - rn));
      maxerr_tr = fmax(maxerr_tr, fabs(D[m * N + n] - tr));
      maxerr_exact = fmax(maxerr_exact, fabs(D[m * N + n] - ex));
    }
  printf("N=%3d tf32-valued inputs=%d: max|D - ref(tf32 RN inputs)| = %.3e, max|D - ref(tf32 trunc inputs)| = %.3e, "
         "max|D - fp32 exact| = %.3e\n",
         N, (int)tf32_inputs, maxerr_rn, maxerr_tr, maxerr_exact);
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dD);
  return 0;
}

template <int N>
int check_ts() {
  std::vector<float> A(128 * 32), B(N * 32), D(128 * N);
  srand(7 + N);
  for (auto& a : A) a = tf32_round_host((rand() % 2001 - 1000) / 997.0f, true);
  for (auto& b : B) b = tf32_round_host((rand() % 2001 - 1000) / 991.0f, true);
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4);
  cudaMalloc(&dB, B.size() * 4);
  cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  const int smem = 1024 + N * 128;
  cudaFuncSetAttribute(gemm_once_ts<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  gemm_once_ts<N><<<1, 128, smem>>>(dA, dB, dD);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("TS N=%d: CUDA error %s\n", N, cudaGetErrorString(e)); return 1; }
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  double maxerr = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < N; ++n) {
      double ex = 0;
      for (int k = 0; k < 32; ++k) ex += (double)A[m * 32 + k] * B[n * 32 + k];
      maxerr = fmax(maxerr, fabs(D[m * N + n] - ex));
    }
  printf("TS N=%3d: max|D - exact| = %.3e  (D[0][0]=%f)\n", N, maxerr, D[0]);
  cudaFree(dA); cudaFree(dB); cudaFree(dD);
  return maxerr > 1e-4;
}

template <int N>
void rate_ts(int sms) {
  float* sink;
  cudaMalloc(&sink, 4 * 1024);
  const int smem = 1024 + N * 128;
  cudaFuncSetAttribute(mma_rate_ts<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 4000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  mma_rate_ts<N><<<sms, 128, smem>>>(100, sink);
  cudaEventRecord(e0);
  mma_rate_ts<N><<<sms, 128, smem>>>(iters, sink);
  cudaEventRecord(e1);
  cudaError_t err = cudaEventSynchronize(e1);
  if (err != cudaSuccess) { printf("rate_ts N=%d: %s\n", N, cudaGetErrorString(err)); exit(1); }
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flops = 2.0 * 128 * N * 32 * (double)iters * sms;
  printf("tf32 MMA TS M=128 N=%3d K=8 (A in TMEM, 1 CTA/SM x %d): %.3f ms  %.1f TFLOP/s\n", N, sms, ms, flops / ms / 1e9);
  cudaFree(sink);
}

void tmem_rate(int sms, int warps, int do_store) {
  float* sink;
  cudaMalloc(&sink, 4);
  const int iters = 20000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  tmem_bw<<<sms, 32 * warps>>>(10, do_store, sink);
  cudaEventRecord(e0);
  tmem_bw<<<sms, 32 * warps>>>(iters, do_store, sink);
  cudaEventRecord(e1);
  cudaError_t err = cudaEventSynchronize(e1);
  if (err != cudaSuccess) { printf("tmem_bw: %s\n", cudaGetErrorString(err)); exit(1); }
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double bytes = (double)sms * warps * 32 * 64 * 4 * iters * (do_store ? 2 : 1);
  const double cycles = ms * 1e-3 * 1.965e9;
  printf("TMEM %s %d warps/SM: %.3f ms  %.1f B/cycle/SM\n", do_store ? "ld+st" : "ld", warps, ms, bytes / sms / cycles);
  cudaFree(sink);
}

template <int N>
void rate(int sms) {
  float* sink;
  cudaMalloc(&sink, 4 * 1024);
  const int smem = 1024 + (128 + N) * 128;
  cudaFuncSetAttribute(mma_rate<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 4000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  mma_rate<N><<<sms, 128, smem>>>(100, sink);
  cudaEventRecord(e0);
  mma_rate<N><<<sms, 128, smem>>>(iters, sink);
  cudaEventRecord(e1);
  cudaError_t err = cudaEventSynchronize(e1);
  if (err != cudaSuccess) { printf("rate N=%d: %s\n", N, cudaGetErrorString(err)); exit(1); }
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flops = 2.0 * 128 * N * 32 * (double)iters * sms;
  printf("tf32 MMA M=128 N=%3d K=8 (SS, 1 CTA/SM x %d): %.3f ms  %.1f TFLOP/s\n", N, sms, ms, flops / ms / 1e9);
  cudaFree(sink);
}

// Sustained rate: the N = 256 SS loop launched back to back for ~4 s (the
// regime of a long GEMM under the board power limit; MEASURED_PEAKS.json's
// bf16 "sustained" figure is measured the same way).  Reports the median of
// the last second's launches and the median SM clock sampled by nvidia-smi
// is left to the caller.
template <int N>
void rate_sustained(int sms, double seconds) {
  float* sink;
  cudaMalloc(&sink, 4 * 1024);
  const int smem = 1024 + (128 + N) * 128;
  cudaFuncSetAttribute(mma_rate<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 4000;
  const double flops = 2.0 * 128 * N * 32 * (double)iters * sms;
  std::vector<float> ms_all;
  double total = 0;
  while (total < seconds * 1e3) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    mma_rate<N><<<sms, 128, smem>>>(iters, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms_all.push_back(ms);
    total += ms;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  }
  std::vector<float> tail(ms_all.end() - ms_all.size() / 4, ms_all.end());
  std::sort(tail.begin(), tail.end());
  const float med = tail[tail.size() / 2];
  printf("tf32 MMA M=128 N=%3d K=8 (SS) sustained %.1f s: last-quarter median %.3f ms  %.1f TFLOP/s\n", N,
         total / 1e3, med, flops / med / 1e9);
  cudaFree(sink);
}

int main(int argc, char** argv) {
  setvbuf(stdout, nullptr, _IONBF, 0);
  if (argc > 1 && std::string(argv[1]) == "--sustained") {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    rate_sustained<256>(sms, 4.0);
    return 0;
  }
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int bad = 0;
  bad |= check<64>(true);
  bad |= check<128>(true);
  bad |= check<256>(true);
  bad |= check<128>(false);  // raw fp32 inputs: does the tensor core truncate or round?
  if (bad) return 1;
  if (check_ts<64>() | check_ts<128>()) return 1;
  rate_ts<64>(sms);
  rate_ts<128>(sms);
  rate_ts<256>(sms);
  tmem_rate(sms, 4, 0);
  tmem_rate(sms, 8, 0);
  tmem_rate(sms, 4, 1);
  tmem_rate(sms, 8, 1);
  rate<64>(sms);
  rate<128>(sms);
  rate<256>(sms);
  return 0;
}
