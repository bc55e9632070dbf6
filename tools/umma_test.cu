// tcgen05 (UMMA) bring-up test: C (M x N, fp32) = A (M x K) . B (N x K)^T with bf16 operands in
// shared memory in the canonical K-major, no-swizzle layout, accumulator in TMEM, read back with
// tcgen05.ld.  Checked against a host reference on the same bf16-rounded inputs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/umma_test tools/umma_test.cu
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

constexpr int M = 128, N = 128, K = 64;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// canonical K-major no-swizzle: element (r, k) at (r/8)*SBO + (k/8)*LBO + (r%8)*16 + (k%8)*2 bytes
__host__ __device__ constexpr uint32_t kmaj_off(int r, int k, uint32_t lbo, uint32_t sbo) {
  return (r / 8) * sbo + (k / 8) * lbo + (r % 8) * 16 + (k % 8) * 2;
}

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;              // descriptor version 1 (sm_100)
  // base offset 0, lbo mode 0, layout type 0 = SWIZZLE_NONE
  return d;
}

__device__ __forceinline__ uint32_t make_idesc_bf16(int m, int n) {
  uint32_t d = 0;
  d |= 1u << 4;                        // c_format = F32
  d |= 1u << 7;                        // a_format = BF16
  d |= 1u << 10;                       // b_format = BF16
  // a_major = b_major = 0 (K-major)
  d |= (uint32_t)(n >> 3) << 17;
  d |= (uint32_t)(m >> 4) << 24;
  return d;
}

__global__ void umma_kernel(const __nv_bfloat16* A, const __nv_bfloat16* B, float* C, int lbo_mode) {
  __shared__ __align__(1024) unsigned char sA[M * K * 2];
  __shared__ __align__(1024) unsigned char sB[N * K * 2];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // operands: LBO (K direction) and SBO (M/N direction), or swapped (lbo_mode 1) to probe the convention
  const uint32_t lbo = 128, sbo = (K / 8) * 128;
  for (int e = tid; e < M * K; e += blockDim.x) {
    const int r = e / K, k = e % K;
    *reinterpret_cast<__nv_bfloat16*>(sA + kmaj_off(r, k, lbo, sbo)) = A[e];
  }
  for (int e = tid; e < N * K; e += blockDim.x) {
    const int r = e / K, k = e % K;
    *reinterpret_cast<__nv_bfloat16*>(sB + kmaj_off(r, k, lbo, sbo)) = B[e];
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base)),
                 "r"(N));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&mbar)));
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");   // generic smem writes -> async proxy
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = tmem_base;
  if (tid == 0) {
    const uint32_t idesc = make_idesc_bf16(M, N);
    const uint32_t l = lbo_mode ? sbo : lbo, s = lbo_mode ? lbo : sbo;
    for (int kk = 0; kk < K / 16; ++kk) {
      // K step of 16 = two core matrices along K
      const uint64_t da = make_desc(smem_u32(sA) + kk * 2 * lbo, l, s);
      const uint64_t db = make_desc(smem_u32(sB) + kk * 2 * lbo, l, s);
      const uint32_t acc = kk > 0 ? 1u : 0u;
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
          "l"(da), "l"(db), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
        smem_u32(&mbar)));
  }
  // wait for the MMAs (phase 0)
  {
    uint32_t done = 0;
    while (!done) {
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
          : "=r"(done)
          : "r"(smem_u32(&mbar)), "r"(0));
    }
  }
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  // TMEM -> registers: warp w reads lanes 32w..32w+31 (rows), 16 columns per load
  const int row = warp * 32 + lane;
  for (int c0 = 0; c0 < N; c0 += 16) {
    uint32_t v[16];
    const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + c0;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
    for (int j = 0; j < 16; ++j) C[row * N + c0 + j] = __uint_as_float(v[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(N));
}

int main() {
  std::vector<__nv_bfloat16> A(M * K), B(N * K);
  std::vector<float> Af(M * K), Bf(N * K);
  uint64_t s = 12345;
  auto rnd = [&]() { s ^= s << 13; s ^= s >> 7; s ^= s << 17; return (double)(s >> 11) * 0x1p-53 - 0.5; };
  for (int i = 0; i < M * K; ++i) { A[i] = __float2bfloat16((float)rnd()); Af[i] = __bfloat162float(A[i]); }
  for (int i = 0; i < N * K; ++i) { B[i] = __float2bfloat16((float)rnd()); Bf[i] = __bfloat162float(B[i]); }
  __nv_bfloat16 *dA, *dB; float* dC;
  cudaMalloc(&dA, A.size() * 2); cudaMalloc(&dB, B.size() * 2); cudaMalloc(&dC, M * N * 4);
  cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice);
  for (int mode = 0; mode < 2; ++mode) {
    cudaMemset(dC, 0, M * N * 4);
    umma_kernel<<<1, 128>>>(dA, dB, dC, mode);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> C(M * N);
    cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0.0, maxref = 0.0;
    for (int i = 0; i < M; ++i)
      for (int j = 0; j < N; ++j) {
        double r = 0.0;
        for (int k = 0; k < K; ++k) r += (double)Af[i * K + k] * Bf[j * K + k];
        maxerr = fmax(maxerr, fabs(r - C[i * N + j]));
        maxref = fmax(maxref, fabs(r));
      }
    printf("lbo_mode %d: %s  max|C - ref| = %.3e (max|ref| %.3e)  C[0..3] %g %g %g %g\n", mode, cudaGetErrorString(e),
           maxerr, maxref, C[0], C[1], C[2], C[3]);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
