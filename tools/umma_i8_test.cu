// tcgen05 kind::i8 bring-up: C (M x N, s32) = A (M x K, s8) . B (N x K, s8)^T, canonical K-major
// no-swizzle operands (8-row x 16-byte core matrices), checked exactly against a host reference.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/umma_i8_test tools/umma_i8_test.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

constexpr int M = 128, K = 64;
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__host__ __device__ constexpr uint32_t kmaj8(int r, int k, uint32_t sbo) {   // int8: core matrix 8 rows x 16 B
  return (r / 8) * sbo + (k / 16) * 128 + (r % 8) * 16 + (k % 16);
}
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
__device__ __forceinline__ uint32_t idesc_i8(int m, int n) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

template <int N>
__global__ void kern(const int8_t* A, const int8_t* B, int32_t* C) {
  __shared__ __align__(1024) int8_t sA[M * K];
  __shared__ __align__(1024) int8_t sB[N * K];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t sbo = (K / 16) * 128;
  for (int e = tid; e < M * K; e += blockDim.x) sA[kmaj8(e / K, e % K, sbo)] = A[e];
  for (int e = tid; e < N * K; e += blockDim.x) sB[kmaj8(e / K, e % K, sbo)] = B[e];
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
  if (tid == 0) {
    for (int kk = 0; kk < K / 32; ++kk) {   // K = 32 per MMA: two 16-byte core matrices
      const uint64_t da = desc(smem_u32(sA) + kk * 256, 128, sbo), db = desc(smem_u32(sB) + kk * 256, 128, sbo);
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
                   "l"(da), "l"(db), "r"(idesc_i8(M, N)), "r"(kk));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&bar)));
  }
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
                 : "=r"(done) : "r"(smem_u32(&bar)) : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const int row = warp * 32 + lane;
  for (int c0 = 0; c0 < N; c0 += 16) {
    uint32_t v[16];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                   "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                 : "r"(tmem + ((uint32_t)(warp * 32) << 16) + c0));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
    for (int j = 0; j < 16; ++j) C[row * N + c0 + j] = (int32_t)v[j];
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(256));
}

template <int N>
int check() {
  std::vector<int8_t> A(M * K), B(N * K);
  uint64_t s = 99;
  auto rnd = [&]() { s ^= s << 13; s ^= s >> 7; s ^= s << 17; return (int8_t)((int)(s % 255) - 127); };
  for (auto& x : A) x = rnd();
  for (auto& x : B) x = rnd();
  int8_t *dA, *dB; int32_t* dC;
  cudaMalloc(&dA, A.size()); cudaMalloc(&dB, B.size()); cudaMalloc(&dC, M * N * 4);
  cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
  kern<N><<<1, 128>>>(dA, dB, dC);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<int32_t> C(M * N);
  cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost);
  long bad = 0;
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j) {
      int32_t r = 0;
      for (int k = 0; k < K; ++k) r += (int32_t)A[i * K + k] * B[j * K + k];
      bad += (r != C[i * N + j]);
    }
  printf("kind::i8 M=%d N=%d K=%d: %s, mismatches %ld (C[0] %d)\n", M, N, K, cudaGetErrorString(e), bad, C[0]);
  return bad != 0 || e != cudaSuccess;
}

int main() { return check<64>() | check<256>(); }
