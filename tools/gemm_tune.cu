// Tuning harness for the dense DMMA GEMM (gemm_dense.cuh) at the cfg3 shape:
// W = A X, A 32768 x 32768, X 32768 x 64 (FP64).  Prints TFLOP/s per tile variant / split.
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
#include "../paper_2602_23778_b200/csrc/gemm_dense.cuh"
using namespace rf;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); return; } } while (0)

__global__ void fill(double* p, size_t n, unsigned seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    unsigned x = (unsigned)(i * 2654435761u) ^ seed;
    x ^= x >> 13; x *= 0x5bd1e995; x ^= x >> 15;
    p[i] = (double)(x & 0xffffff) / 16777216.0 - 0.5;
  }
}

template <int NT, int BM, int WM, int WN, int BK, int ST>
void run(const char* name, const double* A, const double* X, double* out, int64_t n, int k, int* status) {
  using C = GemmCfg<NT, BM, WM, WN, BK, ST>;
  auto kern = gemm_ax_kernel<NT, BM, WM, WN, BK, ST>;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, C::THREADS, C::SMEM));
  const int gx = (int)((n + BM - 1) / BM);
  const int64_t kiters = (n + BK - 1) / BK;
  for (int s : {4, 8, 12, 16}) {
    const int64_t kchunk = ((kiters + s - 1) / s) * BK;
    const int ns = (int)((n + kchunk - 1) / kchunk);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    kern<<<dim3(ns, gx), C::THREADS, C::SMEM>>>(A, n, X, k, n, n, kchunk, out, n * k, 1, 1, status, rf::FusedFinish{});
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    const int reps = 5;
    for (int r = 0; r < reps; ++r)
      kern<<<dim3(ns, gx), C::THREADS, C::SMEM>>>(A, n, X, k, n, n, kchunk, out, n * k, 1, 1, status, rf::FusedFinish{});
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
    printf("%-34s occ %d smem %6d thr %4d split %d ctas %5d : %.3f ms  %.2f TFLOP/s\n", name, occ, C::SMEM,
           C::THREADS, ns, gx * ns, ms, 2.0 * n * n * k / (ms * 1e-3) / 1e12);
  }
}

int main() {
  const int64_t n = 32768;
  const int k = 64;
  double *A, *X, *out;
  int* status;
  cudaMalloc(&A, n * n * 8);
  cudaMalloc(&X, n * k * 8);
  cudaMalloc(&out, 8 * n * k * 8);
  cudaMalloc(&status, 4);
  cudaMemset(status, 0, 4);
  fill<<<4096, 256>>>(A, n * n, 1);
  fill<<<4096, 256>>>(X, n * k, 2);
  cudaDeviceSynchronize();
  run<64, 128, 32, 32, 32, 2>("BM128 W32x32 BK32 S2", A, X, out, n, k, status);
  run<64, 128, 32, 32, 16, 3>("BM128 W32x32 BK16 S3", A, X, out, n, k, status);
  run<64, 128, 32, 32, 16, 2>("BM128 W32x32 BK16 S2", A, X, out, n, k, status);
  run<64, 64, 32, 32, 32, 2>("BM64 W32x32 BK32 S2", A, X, out, n, k, status);
  run<64, 128, 16, 32, 32, 2>("BM128 W16x32 BK32 S2 16w", A, X, out, n, k, status);
  run<64, 128, 32, 16, 32, 2>("BM128 W32x16 BK32 S2 16w", A, X, out, n, k, status);
  run<64, 192, 32, 32, 16, 2>("BM192 W32x32 BK16 S2 12w", A, X, out, n, k, status);
  run<64, 128, 64, 16, 32, 2>("BM128 W64x16 BK32 S2", A, X, out, n, k, status);
  return 0;
}
