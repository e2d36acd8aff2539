// f16_probe.cu -- can the DWM GEMM run its 3-term split on kind::f16?
//
// (1) layout + rounding: D[128x64] = A[128x256] * B[64x256]^T with fp16 inputs,
//     A resident in TMEM (two fp16 per 32-bit column, even k in the low half),
//     B K-major SW128 in smem; one accumulator over 16 K=16 MMAs and 4 chunk
//     accumulators (4 MMAs each) summed in FP32 RN.  Error vs the exact sum.
// (2) throughput: 148 CTAs, one MMA warp, per 64-channel stage 4 x (N=128 +
//     N=64) kind::f16 TS MMAs (the same N as the tf32 GEMM's 8 x (N=128 + N=64)).
//
//   ./f16_probe
#include <cuda_fp16.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../paper_2002_00552_b200/csrc/dwm_sm100.cuh"
using namespace dwm::sm100;

constexpr int N = 64, K = 256;

// byte offset of (row r, byte kb) in a K-major SW128 tile whose rows are 128 bytes
__device__ __forceinline__ uint32_t sw128_byte(uint32_t r, uint32_t kb) {
  return (r >> 3) * 1024u + (r & 7u) * 128u + (((kb >> 4) ^ (r & 7u)) << 4) + (kb & 15u);
}

__global__ void acc_kernel(const __half* A, const __half* B, float* out1, float* out4) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  // B: 4 atoms (64 K each) of [64 rows][128 B]
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid / 32;
  for (int e = tid; e < N * K; e += blockDim.x) {
    const int r = e / K, k = e % K;
    *(__half*)(smem + (k / 64) * 8192 + sw128_byte(r, (k % 64) * 2)) = B[e];
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
  const uint32_t t = tmem_base;
  const uint32_t la = t + ((uint32_t)(32 * warp) << 16);
  // A rows into TMEM columns 256.. (row = lane), column j = {A[k=2j] lo, A[k=2j+1] hi}
  for (int c0 = 0; c0 < K / 2; c0 += 16) {
    float v[16];
    for (int j = 0; j < 16; ++j) {
      const __half lo = A[tid * K + 2 * (c0 + j)], hi = A[tid * K + 2 * (c0 + j) + 1];
      const uint32_t u = (uint32_t)__half_as_ushort(lo) | ((uint32_t)__half_as_ushort(hi) << 16);
      v[j] = __uint_as_float(u);
    }
    tmem_st16(la + 256 + c0, v);
  }
  tmem_st_wait();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) {
    if (tid == 0) {
      const uint32_t idesc = idesc_f16(128, N);
      for (int kk = 0; kk < K / 16; ++kk) {
        const uint64_t db = sdesc_sw128(smem_u32(smem) + (kk / 4) * 8192 + 32 * (kk % 4));
        mma_f16_ts(t, t + 256 + 8 * kk, db, idesc, kk != 0);                          // single accumulator
        mma_f16_ts(t + 64 + 64 * (kk / 4), t + 256 + 8 * kk, db, idesc, (kk % 4) != 0);  // 4 chunk accumulators
      }
      mma_commit(&bar);
    }
    __syncwarp();
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  for (int c0 = 0; c0 < N; c0 += 16) {
    float v[16];
    tmem_ld16(la + c0, v);
    tmem_ld_wait();
    for (int j = 0; j < 16; ++j) out1[tid * N + c0 + j] = v[j];
    float s[16];
    for (int j = 0; j < 16; ++j) s[j] = 0.f;
    for (int ch = 0; ch < 4; ++ch) {
      tmem_ld16(la + 64 + 64 * ch + c0, v);
      tmem_ld_wait();
      for (int j = 0; j < 16; ++j) s[j] = __fadd_rn(s[j], v[j]);
    }
    for (int j = 0; j < 16; ++j) out4[tid * N + c0 + j] = s[j];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(t);
}

// throughput: kind 0 = f16 (4 K=16 steps per stage), 1 = tf32 (8 K=8 steps)
__global__ void rate_kernel(int iters, int kind, long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t done[4];
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid / 32;
  for (int e = tid; e < 3 * 2 * 16384 / 4; e += blockDim.x) ((float*)smem)[e] = 0.f;
  if (tid == 0) {
    for (int i = 0; i < 4; ++i) mbar_init(&done[i], 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(&tmem_base);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t t = tmem_base;
  if (warp == 0) {
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const int sb = it % 3;
      const uint32_t dacc = t + 128 * (it & 1), a = t + 256 + 128 * (it & 1);
      if (elect_one()) {
        if (kind == 0) {
          const uint32_t i128 = idesc_f16(128, 128), i64 = idesc_f16(128, 64);
          const uint64_t du = sdesc_sw128(smem_u32(smem + sb * 2 * 16384));
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            mma_f16_ts(dacc, a + 8 * kk, du + 2 * kk, i128, kk != 0);
            mma_f16_ts(dacc + 64, a + 32 + 8 * kk, du + 2 * kk, i64, 1u);
          }
        } else {
          const uint32_t i128 = idesc_tf32(128, 128), i64 = idesc_tf32(128, 64);
          for (int h = 0; h < 2; ++h) {
            const uint64_t du = sdesc_sw128(smem_u32(smem + (sb * 2 + h) * 16384));
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              mma_tf32_ts(dacc, a + 32 * h + 8 * kk, du + 2 * kk, i128, (h == 0 && kk == 0) ? 0u : 1u);
              mma_tf32_ts(dacc + 64, a + 64 + 32 * h + 8 * kk, du + 2 * kk, i64, 1u);
            }
          }
        }
        mma_commit(&done[it % 4]);
      }
      __syncwarp();
      if (it >= 1) mbar_wait(&done[(it - 1) % 4], ((it - 1) / 4) & 1);
    }
    mbar_wait(&done[(iters - 1) % 4], ((iters - 1) / 4) & 1);
    if (tid == 0) cyc[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(t);
}

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  for (int mode = 0; mode < 2; ++mode) {
    std::vector<__half> A(128 * K), B(N * K);
    std::vector<float> Af(128 * K), Bf(N * K), D1(128 * N), D4(128 * N);
    srand(3 + mode);
    for (size_t i = 0; i < A.size(); ++i) {
      A[i] = __float2half((rand() / (float)RAND_MAX) * (mode ? 2.f : 1.f) - (mode ? 1.f : 0.f));
      Af[i] = __half2float(A[i]);
    }
    for (size_t i = 0; i < B.size(); ++i) {
      B[i] = __float2half((rand() / (float)RAND_MAX) * (mode ? 2.f : 1.f) - (mode ? 1.f : 0.f));
      Bf[i] = __half2float(B[i]);
    }
    __half *dA, *dB;
    float *d1, *d4;
    cudaMalloc(&dA, A.size() * 2);
    cudaMalloc(&dB, B.size() * 2);
    cudaMalloc(&d1, D1.size() * 4);
    cudaMalloc(&d4, D4.size() * 4);
    cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice);
    const int smem = 1024 + 4 * 8192;
    cudaFuncSetAttribute(acc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    acc_kernel<<<1, 128, smem>>>(dA, dB, d1, d4);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("error %s\n", cudaGetErrorString(e));
      return 1;
    }
    cudaMemcpy(D1.data(), d1, D1.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(D4.data(), d4, D4.size() * 4, cudaMemcpyDeviceToHost);
    double s1 = 0, q1 = 0, s4 = 0, q4 = 0, sf = 0, qf = 0, mx = 0;
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < N; ++n) {
        double ex = 0;
        float seq = 0.f;
        for (int k = 0; k < K; ++k) {
          ex += (double)Af[m * K + k] * Bf[n * K + k];
          seq = fmaf(Af[m * K + k], Bf[n * K + k], seq);
        }
        const double ulp = ldexp(1.0, ilogb(fabs(ex)) - 23);
        const double e1 = (D1[m * N + n] - ex) / ulp, e4 = (D4[m * N + n] - ex) / ulp, ef = (seq - ex) / ulp;
        s1 += e1; q1 += e1 * e1; s4 += e4; q4 += e4 * e4; sf += ef; qf += ef * ef;
        mx = fmax(mx, fabs(e1));
      }
    const double cnt = 128.0 * N;
    printf("%s inputs: single TMEM acc (16 K=16 MMAs): mean %+.3f ulp rms %.3f max %.1f | 4 chunk accs + fp32 RN: mean %+.3f rms %.3f | "
           "sequential fp32 FMA: mean %+.3f rms %.3f\n",
           mode ? "signed  " : "positive", s1 / cnt, sqrt(q1 / cnt), mx, s4 / cnt, sqrt(q4 / cnt), sf / cnt, sqrt(qf / cnt));
  }
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* cyc;
  cudaMalloc(&cyc, sizeof(long long) * sms);
  const int smem = 1024 + 3 * 2 * 16384;
  cudaFuncSetAttribute(rate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int kind = 0; kind < 2; ++kind) {
    const int iters = 4000;
    rate_kernel<<<sms, 128, smem>>>(10, kind, cyc);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    rate_kernel<<<sms, 128, smem>>>(iters, kind, cyc);
    cudaEventRecord(e1);
    if (cudaEventSynchronize(e1) != cudaSuccess) {
      printf("kind %d: error %s\n", kind, cudaGetErrorString(cudaGetLastError()));
      return 1;
    }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    long long c0;
    cudaMemcpy(&c0, cyc, sizeof(c0), cudaMemcpyDeviceToHost);
    const double flops = 2.0 * 128 * 192 * 64 * (double)iters * sms;  // per 64-channel stage, N = 128 + 64
    printf("%s: %.1f cycles per 64-channel stage, %.1f TFLOP/s (N=192 per K)\n", kind ? "tf32" : "f16 ",
           (double)c0 / iters, flops / ms / 1e9);
  }
  return 0;
}
