// FP64-accurate A X on the INT8 tensor cores (ozaki.cuh) vs the DMMA GEMM (gemm_dense.cuh) at the
// cfg3 shape: accuracy against sum_l |A_il||X_lj| and timing.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/oz_test tools/oz_test.cu
#include <cstdio>
#include <cmath>
#include <vector>
#include <climits>
#include <cuda_runtime.h>
#include "../paper_2602_23778_b200/csrc/gemm_dense.cuh"
#include "../paper_2602_23778_b200/csrc/ozaki.cuh"
using namespace rf;

__global__ void fill(double* p, int64_t n, uint64_t seed, double scale) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t z = (i + 1) * 0x9E3779B97F4A7C15ull ^ seed;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull; z = (z ^ (z >> 27)) * 0x94D049BB133111EBull; z ^= z >> 31;
    p[i] = ((double)(z >> 11) * 0x1p-53 - 0.5) * scale;
  }
}
__global__ void absgemm(const double* A, const double* X, int64_t n, int k, double* B, int rows) {  // sample rows
  const int j = threadIdx.x;
  const int64_t i = (int64_t)blockIdx.x * (n / rows);
  double s = 0.0;
  for (int64_t l = 0; l < n; ++l) s += fabs(A[i * n + l]) * fabs(X[l * k + j]);
  B[blockIdx.x * k + j] = s;
}

int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? atoll(argv[1]) : 32768;
  constexpr int k = 64;
  const int sms = 148;
  double *A, *X, *W1, *W2, *Ab, *dg; int *st; int32_t *e, *f; int8_t *As, *Xs;
  cudaMalloc(&A, n * n * 8); cudaMalloc(&X, n * k * 8); cudaMalloc(&st, 4); cudaMemset(st, 0, 4);
  fill<<<4096, 256>>>(A, n * n, 1, 2.0); fill<<<1184, 256>>>(X, n * k, 2, 0.02);
  const int64_t nks = (n + OZ_BK - 1) / OZ_BK, nrt = (n + OZ_BM - 1) / OZ_BM;
  cudaMalloc(&e, n * 4); cudaMalloc(&f, k * 4); cudaMalloc(&dg, n * 8);
  cudaMalloc(&As, nrt * nks * OZ_S * (int64_t)OZ_ATILE); cudaMalloc(&Xs, nks * OZ_S * (int64_t)k * OZ_BK);
  // DMMA reference (split 4)
  using GC = GemmCfg<64, 128, 64, 16, 32, 2>;
  auto g = gemm_ax_kernel<64, 128, 64, 16, 32, 2>;
  cudaFuncSetAttribute(g, cudaFuncAttributeMaxDynamicSharedMemorySize, GC::SMEM);
  const int ns = 4;
  const int64_t kchunk = (n / ns + 31) / 32 * 32;
  cudaMalloc(&W1, ns * n * k * 8); cudaMalloc(&W2, ns * n * k * 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  g<<<dim3(ns, (n + 127) / 128), GC::THREADS, GC::SMEM>>>(A, n, X, k, n, n, kchunk, W1, n * k, 1, 1, st, rf::FusedFinish{});
  cudaEventRecord(a);
  g<<<dim3(ns, (n + 127) / 128), GC::THREADS, GC::SMEM>>>(A, n, X, k, n, n, kchunk, W1, n * k, 1, 1, st, rf::FusedFinish{});
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms1; cudaEventElapsedTime(&ms1, a, b);
  // init slicing
  cudaEventRecord(a);
  oz_rowexp_kernel<<<sms * 8, 256>>>(A, n, n, n, 0, e, dg);
  oz_slice_A_kernel<<<sms * 16, 256>>>(A, n, n, n, 0, e, As, nks);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float msi; cudaEventElapsedTime(&msi, a, b);
  printf("init slicing: %.3f ms (%s)\n", msi, cudaGetErrorString(cudaGetLastError()));
  // per sweep
  using OC = OzCfg<k>;
  cudaFuncSetAttribute(oz_gemm_kernel<k>, cudaFuncAttributeMaxDynamicSharedMemorySize, OC::SMEM);
  const int64_t ks_per = (nks + ns - 1) / ns;
  auto sweep = [&]() {
    cudaMemsetAsync(f, 0x80, k * 4);
    oz_colexp_kernel<<<sms * 4, 256>>>(X, n, k, f);
    oz_slice_X_kernel<<<sms * 8, 256>>>(X, n, k, f, Xs, nks);
    oz_gemm_kernel<k><<<dim3(nrt, ns), OZ_THREADS, OC::SMEM>>>(As, Xs, e, f, n, nks, ks_per, W2, n * k, dg, X, 0, st);
  };
  sweep();
  cudaError_t err = cudaDeviceSynchronize();
  printf("first oz sweep: %s\n", cudaGetErrorString(err));
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) sweep();
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms2; cudaEventElapsedTime(&ms2, a, b);
  ms2 /= 5;
  cudaEventRecord(a);
  oz_gemm_kernel<k><<<dim3(nrt, ns), OZ_THREADS, OC::SMEM>>>(As, Xs, e, f, n, nks, ks_per, W2, n * k, dg, X, 0, st);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms3; cudaEventElapsedTime(&ms3, a, b);
  // compare sums of splits on sampled rows
  const int rows = 64;
  cudaMalloc(&Ab, rows * k * 8);
  absgemm<<<rows, k>>>(A, X, n, k, Ab, rows);
  std::vector<double> w1(ns * n * k), w2(ns * n * k), ab(rows * k);
  cudaMemcpy(w1.data(), W1, w1.size() * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(w2.data(), W2, w2.size() * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(ab.data(), Ab, ab.size() * 8, cudaMemcpyDeviceToHost);
  double worst = 0, worstall = 0;
  for (int q = 0; q < rows; ++q)
    for (int j = 0; j < k; ++j) {
      const int64_t i = (int64_t)q * (n / rows);
      double s1 = 0, s2 = 0;
      for (int s = 0; s < ns; ++s) { s1 += w1[s * n * k + i * k + j]; s2 += w2[s * n * k + i * k + j]; }
      worst = fmax(worst, fabs(s1 - s2) / ab[q * k + j]);
    }
  for (int64_t i = 0; i < n; ++i)
    for (int j = 0; j < k; ++j) {
      double s1 = 0, s2 = 0;
      for (int s = 0; s < ns; ++s) { s1 += w1[s * n * k + i * k + j]; s2 += w2[s * n * k + i * k + j]; }
      worstall = fmax(worstall, fabs(s1 - s2) / fmax(fabs(s1), 1e-300));
    }
  printf("n=%lld k=%d: DMMA gemm %.3f ms (%.1f TF) | oz sweep-side %.3f ms, oz gemm %.3f ms (%.1f TF eq.)\n",
         (long long)n, k, ms1, 2.0 * n * n * k / ms1 / 1e9, ms2, ms3, 2.0 * n * n * k / ms3 / 1e9);
  printf("max |W_oz - W_dmma| / (|A||X|) over %d sampled rows: %.3e   (n u = %.3e); max rel elementwise %.3e\n", rows,
         worst, n * 0x1p-53, worstall);
  return 0;
}
