// FP64 pass B (passB_kernel, 2-D tiles) variants at the cfg4 shape (n = 1,045,504, k = 32).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/passb32_tune tools/passb32_tune.cu
#include <cstdio>
#include <algorithm>
#include <cuda_runtime.h>
#include "../paper_2602_23778_b200/csrc/passes.cuh"
using namespace rf;

__global__ void fill(double* p, int64_t n, uint64_t seed, double scale) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t z = (i + 1) * 0x9E3779B97F4A7C15ull ^ seed;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull; z = (z ^ (z >> 27)) * 0x94D049BB133111EBull; z ^= z >> 31;
    p[i] = ((double)(z >> 11) * 0x1p-53 - 0.5) * scale;
  }
}

template <int TA, int TB, int WA, int WB, int BR>
void run(Ws ws, const double* X, int sms, double* bp) {
  using C = PassBCfg<32, TA, TB, WA, WB, BR>;
  auto k = passB_kernel<32, TA, TB, WA, WB, BR>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, C::THREADS, C::SMEM);
  const int64_t rows = ws.n_loc;
  const int gy = (int)std::min<int64_t>(std::max(sms * occ / C::NTILES, 1), (rows + 255) / 256);
  ws.bpart = bp;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  k<<<dim3(C::NTILES, gy), C::THREADS, C::SMEM>>>(ws, X, 1);
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) k<<<dim3(C::NTILES, gy), C::THREADS, C::SMEM>>>(ws, X, 1);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("TA=%d TB=%d warps %dx%d BR=%d tiles %d occ %d gy %d: %.4f ms  %.1f TF (4nk^2)  %s\n", TA, TB, WA, WB, BR,
         C::NTILES, occ, gy, ms / 5, 4.0 * rows * 32 * 32 / (ms / 5) / 1e9, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const int64_t n = 1045504; const int k = 32, sms = 148;
  double *X, *W, *d, *bp, *brr; int* st;
  cudaMalloc(&X, n * k * 8); cudaMalloc(&W, n * k * 8); cudaMalloc(&d, k * 8); cudaMalloc(&st, 4);
  cudaMalloc(&bp, (size_t)64 << 20); cudaMalloc(&brr, (size_t)8 << 20);
  cudaMemset(st, 0, 4);
  fill<<<1184, 256>>>(X, n * k, 1, 1e-3); fill<<<1184, 256>>>(W, n * k, 2, 1e-3); fill<<<1, 64>>>(d, k, 3, 1.0);
  Ws ws{};
  ws.n_loc = n; ws.k = k; ws.kp = 32; ws.top = 0; ws.W = W; ws.d = d; ws.status = st; ws.brr = brr;
  run<32, 64, 2, 4, 32>(ws, X, sms, bp);
  run<32, 64, 2, 2, 32>(ws, X, sms, bp);
  run<32, 64, 1, 4, 32>(ws, X, sms, bp);
  run<32, 64, 2, 2, 16>(ws, X, sms, bp);
  run<32, 64, 1, 4, 16>(ws, X, sms, bp);
  run<32, 64, 2, 2, 8>(ws, X, sms, bp);
  run<32, 64, 4, 1, 32>(ws, X, sms, bp);
  run<32, 64, 4, 2, 32>(ws, X, sms, bp);
  return 0;
}
