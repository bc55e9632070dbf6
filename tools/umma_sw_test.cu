// tcgen05 bring-up, 128B-swizzled K-major operands: C (M x N, fp32) = A (M x K) . B (N x K)^T,
// K = 128 as two 64-wide swizzle atoms, K steps of 16 advance the descriptor start by 32 B inside
// an atom.  Also times a long chain of M = 128, N = 16 MMAs in both layouts (SMEM A-read rate).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/umma_sw_test tools/umma_sw_test.cu
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

constexpr int M = 128, N = 128, K = 128;
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// 128B swizzle, K-major: element (r, k) of an R-row operand
__host__ __device__ constexpr uint32_t sw128_off(int r, int k, int R) {
  return (uint32_t)(k / 64) * (R * 128) + (r / 8) * 1024 + (r % 8) * 128 + ((((k % 64) / 8) ^ (r % 8)) * 16) + (k % 8) * 2;
}
__host__ __device__ constexpr uint32_t kmaj_off(int r, int k, uint32_t sbo) {
  return (r / 8) * sbo + (k / 8) * 128 + (r % 8) * 16 + (k % 8) * 2;
}
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;                  // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;        // SBO: 8-row groups 1024 B apart
  d |= (uint64_t)1 << 46;                  // version
  d |= (uint64_t)2 << 61;                  // SWIZZLE_128B
  return d;
}
__device__ __forceinline__ uint64_t desc_none(uint32_t saddr, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)(128 >> 4) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
__device__ __forceinline__ uint32_t idesc_bf16(int m, int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}
__device__ __forceinline__ void mma(uint32_t tmem, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
               "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void wait_bar(uint64_t* bar, uint32_t par) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
                 : "=r"(done) : "r"(smem_u32(bar)), "r"(par) : "memory");
}

__global__ void kern(const __nv_bfloat16* A, const __nv_bfloat16* B, float* C, int mode, int reps, long long* cyc) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* sA = sm;                 // 32 KB
  unsigned char* sB = sm + M * K * 2;     // 32 KB
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int e = tid; e < M * K; e += blockDim.x) {
    const int r = e / K, k = e % K;
    const uint32_t oa = mode ? sw128_off(r, k, M) : kmaj_off(r, k, (K / 8) * 128);
    *reinterpret_cast<__nv_bfloat16*>(sA + oa) = A[e];
  }
  for (int e = tid; e < N * K; e += blockDim.x) {
    const int r = e / K, k = e % K;
    const uint32_t ob = mode ? sw128_off(r, k, N) : kmaj_off(r, k, (K / 8) * 128);
    *reinterpret_cast<__nv_bfloat16*>(sB + ob) = B[e];
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tbase)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar)));
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = tbase;
  auto dA = [&](int kk) -> uint64_t {
    return mode ? desc_sw128(smem_u32(sA) + (kk / 4) * (M * 128) + (kk % 4) * 32) : desc_none(smem_u32(sA) + kk * 256, (K / 8) * 128);
  };
  auto dB = [&](int kk, int rows) -> uint64_t {
    return mode ? desc_sw128(smem_u32(sB) + (kk / 4) * (rows * 128) + (kk % 4) * 32) : desc_none(smem_u32(sB) + kk * 256, (K / 8) * 128);
  };
  if (tid == 0) {
    for (int kk = 0; kk < K / 16; ++kk) mma(tmem, dA(kk), dB(kk, N), idesc_bf16(M, N), kk > 0);
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&bar)));
  }
  wait_bar(&bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const int row = warp * 32 + lane;
  for (int c0 = 0; c0 < N; c0 += 16) {
    uint32_t v[16];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                   "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                 : "r"(tmem + ((uint32_t)(warp * 32) << 16) + c0));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
    for (int j = 0; j < 16; ++j) C[row * N + c0 + j] = __uint_as_float(v[j]);
  }
  // timing: reps x 8 MMAs of M = 128, N = 16 (B = the first 16 rows of sB: valid for both layouts
  // since the swizzle atom's rows 0-15 are the first two 8-row groups)
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  if (tid == 0) {
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r)
      for (int kk = 0; kk < K / 16; ++kk) {
        uint64_t db = mode ? desc_sw128(smem_u32(sB) + (kk / 4) * (N * 128) + (kk % 4) * 32) : dB(kk, N);
        mma(tmem + 128 + 16 * (r & 7), dA(kk), db, idesc_bf16(M, 16), kk > 0);
      }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&bar)));
    wait_bar(&bar, 1);
    cyc[mode] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(256));
}

int main() {
  std::vector<__nv_bfloat16> A(M * K), B(N * K);
  std::vector<float> Af(M * K), Bf(N * K);
  uint64_t s = 12345;
  auto rnd = [&]() { s ^= s << 13; s ^= s >> 7; s ^= s << 17; return (double)(s >> 11) * 0x1p-53 - 0.5; };
  for (int i = 0; i < M * K; ++i) { A[i] = __float2bfloat16((float)rnd()); Af[i] = __bfloat162float(A[i]); }
  for (int i = 0; i < N * K; ++i) { B[i] = __float2bfloat16((float)rnd()); Bf[i] = __bfloat162float(B[i]); }
  __nv_bfloat16 *dA, *dB; float* dC; long long* dcyc;
  cudaMalloc(&dA, A.size() * 2); cudaMalloc(&dB, B.size() * 2); cudaMalloc(&dC, M * N * 4); cudaMalloc(&dcyc, 16);
  cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * M * K * 2 + 1024);
  const int reps = 512;
  for (int mode = 0; mode < 2; ++mode) {
    cudaMemset(dC, 0, M * N * 4);
    kern<<<1, 128, 2 * M * K * 2 + 1024>>>(dA, dB, dC, mode, reps, dcyc);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> C(M * N);
    long long cyc[2];
    cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(cyc, dcyc, 16, cudaMemcpyDeviceToHost);
    double maxerr = 0.0, maxref = 0.0;
    for (int i = 0; i < M; ++i)
      for (int j = 0; j < N; ++j) {
        double r = 0.0;
        for (int k = 0; k < K; ++k) r += (double)Af[i * K + k] * Bf[j * K + k];
        maxerr = fmax(maxerr, fabs(r - C[i * N + j]));
        maxref = fmax(maxref, fabs(r));
      }
    printf("%s: %s  max|C - ref| = %.3e (max|ref| %.3e)  N=16 MMA: %.1f cycles each\n", mode ? "SW128" : "no-swizzle",
           cudaGetErrorString(e), maxerr, maxref, (double)cyc[mode] / (reps * 8));
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
