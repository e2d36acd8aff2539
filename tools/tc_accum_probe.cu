// tc_accum_probe.cu -- how does the tcgen05 kind::tf32 FP32 accumulator round?
// D = sum_k A[m][k] B[n][k] over K = 256 with tf32-exact inputs, accumulated
// (1) in one TMEM accumulator over 32 K=8 MMAs, (2) in 8 accumulators of 4 MMAs
// each summed on the CUDA cores in FP32 RN.  Compares the signed and RMS error
// against an exact (double) sum and against a sequential FP32 RN FMA chain.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include "../paper_2002_00552_b200/csrc/dwm_sm100.cuh"
using namespace dwm::sm100;

constexpr int N = 64, K = 256, KC = K / 32;

__global__ void acc_kernel(const float* A, const float* B, float* out1, float* out8) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  float* sA = (float*)smem;                       // KC atoms of [128][32]
  float* sB = (float*)(smem + KC * 128 * 128);    // KC atoms of [64][32]
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid / 32;
  for (int e = tid; e < 128 * K; e += blockDim.x) {
    int r = e / K, k = e % K;
    *(float*)((uint8_t*)sA + (k / 32) * 16384 + sw128_offset(r, k % 32)) = A[e];
  }
  for (int e = tid; e < N * K; e += blockDim.x) {
    int r = e / K, k = e % K;
    *(float*)((uint8_t*)sB + (k / 32) * 8192 + sw128_offset(r, k % 32)) = B[e];
  }
  if (tid == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc<512>(&tmem_base);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t t = tmem_base;
  if (warp == 0) {
    if (tid == 0) {
      const uint32_t idesc = idesc_tf32(128, N);
      for (int kc = 0; kc < KC; ++kc)
        for (int k = 0; k < 4; ++k) {
          const uint64_t da = sdesc_sw128(smem_u32(sA) + kc * 16384 + 32 * k);
          const uint64_t db = sdesc_sw128(smem_u32(sB) + kc * 8192 + 32 * k);
          mma_tf32(t, da, db, idesc, (kc | k) != 0);                 // single accumulator
          mma_tf32(t + 64 + 64 * (kc % 7) + (kc / 7) * 0, da, db, idesc, k != 0);  // per-chunk
        }
      mma_commit(&bar);
    }
    __syncwarp();
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  // KC = 8 chunks but only 7 extra slots of 64 cols fit next to the main one: chunk 7 reuses slot 0
  // -> read chunk partials in a second pass is not possible; instead use only chunks 0..6 + recompute 7
  const uint32_t la = t + ((uint32_t)(32 * warp) << 16);
  for (int c0 = 0; c0 < N; c0 += 16) {
    float v[16];
    tmem_ld16(la + c0, v); tmem_ld_wait();
    for (int j = 0; j < 16; ++j) out1[(32 * warp + tid % 32) * N + c0 + j] = v[j];
  }
  for (int c0 = 0; c0 < N; c0 += 16) {
    float s[16];
    for (int j = 0; j < 16; ++j) s[j] = 0.f;
    for (int slot = 0; slot < 7; ++slot) {
      float v[16];
      tmem_ld16(la + 64 + 64 * slot + c0, v); tmem_ld_wait();
      for (int j = 0; j < 16; ++j) s[j] = __fadd_rn(s[j], v[j]);
    }
    for (int j = 0; j < 16; ++j) out8[(32 * warp + tid % 32) * N + c0 + j] = s[j];
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) tmem_dealloc<512>(t);
}

static float tf32r(float x) { uint32_t u; memcpy(&u, &x, 4); u += 0xFFF + ((u >> 13) & 1); u &= 0xFFFFE000u; float r; memcpy(&r, &u, 4); return r; }

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  for (int mode = 0; mode < 2; ++mode) {
    std::vector<float> A(128 * K), B(N * K), D1(128 * N), D8(128 * N);
    srand(3 + mode);
    for (auto& a : A) a = tf32r((rand() / (float)RAND_MAX) * (mode ? 2.f : 1.f) - (mode ? 1.f : 0.f));
    for (auto& b : B) b = tf32r((rand() / (float)RAND_MAX) * (mode ? 2.f : 1.f) - (mode ? 1.f : 0.f));
    float *dA, *dB, *d1, *d8;
    cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&d1, D1.size() * 4); cudaMalloc(&d8, D8.size() * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    const int smem = 1024 + KC * (128 + N) * 128;
    cudaFuncSetAttribute(acc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    acc_kernel<<<1, 128, smem>>>(dA, dB, d1, d8);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    cudaMemcpy(D1.data(), d1, D1.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(D8.data(), d8, D8.size() * 4, cudaMemcpyDeviceToHost);
    double s1 = 0, q1 = 0, s8 = 0, q8 = 0, sf = 0, qf = 0;
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < N; ++n) {
        double ex = 0, ex7 = 0; float seq = 0.f;
        for (int k = 0; k < K; ++k) {
          double p = (double)A[m * K + k] * B[n * K + k];
          ex += p; if (k < 224) ex7 += p;
          seq = fmaf(A[m * K + k], B[n * K + k], seq);
        }
        double ulp = ldexp(1.0, ilogb(fabs(ex)) - 23);
        s1 += (D1[m * N + n] - ex) / ulp; q1 += pow((D1[m * N + n] - ex) / ulp, 2);
        double ulp7 = ldexp(1.0, ilogb(fabs(ex7)) - 23);
        s8 += (D8[m * N + n] - ex7) / ulp7; q8 += pow((D8[m * N + n] - ex7) / ulp7, 2);
        sf += (seq - ex) / ulp; qf += pow((seq - ex) / ulp, 2);
      }
    const double cnt = 128.0 * N;
    printf("%s inputs: single TMEM acc (32 MMAs): mean %+.3f ulp, rms %.3f ulp | 7 chunk accs + fp32 RN sum: mean %+.3f rms %.3f | "
           "sequential fp32 FMA: mean %+.3f rms %.3f\n", mode ? "signed" : "positive",
           s1 / cnt, sqrt(q1 / cnt), s8 / cnt, sqrt(q8 / cnt), sf / cnt, sqrt(qf / cnt));
  }
  return 0;
}
