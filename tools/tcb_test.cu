// passB on tcgen05 (mixed precision) vs the FP64 DMMA pass B2: accuracy of [M2 | G2 | rr2] and timing.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/tcb_test tools/tcb_test.cu
#include <cstdio>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
#include "../paper_2602_23778_b200/csrc/passes.cuh"
#include "../paper_2602_23778_b200/csrc/tc_passes.cuh"
using namespace rf;

__global__ void fill(double* p, int64_t n, uint64_t seed, double scale) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t z = (i + 1) * 0x9E3779B97F4A7C15ull ^ seed;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull; z = (z ^ (z >> 27)) * 0x94D049BB133111EBull; z ^= z >> 31;
    p[i] = ((double)(z >> 11) * 0x1p-53 - 0.5) * scale;
  }
}

int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? atoll(argv[1]) : 4096000;
  const int k = 128, sms = 148;
  double *X, *W, *d, *bp, *brr, *out1, *out2; int* st;
  cudaMalloc(&X, n * k * 8); cudaMalloc(&W, n * k * 8); cudaMalloc(&d, k * 8); cudaMalloc(&st, 4);
  const int chunks = 256;
  cudaMalloc(&bp, (size_t)chunks * 4 * 128 * 64 * 8); cudaMalloc(&brr, (size_t)chunks * 128 * 8);
  double* bd; cudaMalloc(&bd, (size_t)chunks * 2 * 128 * 8);
  cudaMalloc(&out1, (2 * k * k + k) * 8); cudaMalloc(&out2, (2 * k * k + k) * 8);
  fill<<<1184, 256>>>(X, n * k, 1, 1.0 / sqrt((double)n));
  fill<<<1184, 256>>>(W, n * k, 2, 1.0 / sqrt((double)n));
  fill<<<1, 128>>>(d, k, 3, 0.0);   // d = 0: R = W (the mixed pass must still form R exactly)
  cudaMemset(st, 0, 4);
  Ws ws{};
  ws.n_loc = n; ws.k = k; ws.kp = 128; ws.top = 0; ws.W = W; ws.d = d; ws.status = st; ws.bpart = bp; ws.brr = brr;
  // FP64 reference: passB2 (paired grid) + reduce
  using C2 = PassB2Cfg<128>;
  cudaFuncSetAttribute(passB2_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, C2::SMEM);
  const int pairs = 42;
  ws.M2 = out1; ws.G2 = out1 + k * k; ws.rr2 = out1 + 2 * k * k;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  passB2_kernel<128><<<7 * pairs, C2::THREADS, C2::SMEM>>>(ws, X, 1);
  cudaEventRecord(a);
  passB2_kernel<128><<<7 * pairs, C2::THREADS, C2::SMEM>>>(ws, X, 1);
  cudaEventRecord(b);
  passB2_reduce_kernel<128><<<(2 * k * k + k + 31) / 32, PB_RED_THREADS>>>(ws, 2 * pairs);
  cudaEventSynchronize(b);
  float ms1; cudaEventElapsedTime(&ms1, a, b);
  // tcgen05
  cudaFuncSetAttribute(passB_tc_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, TcbCfg<128>::SMEM);
  ws.M2 = out2; ws.G2 = out2 + k * k; ws.rr2 = out2 + 2 * k * k;
  ws.bdiag = bd;   // FP64 diagonals of M2, G2
  passB_tc_kernel<128><<<sms, TCB_THREADS, TcbCfg<128>::SMEM>>>(ws, X);
  cudaError_t e = cudaDeviceSynchronize();
  printf("first tc launch: %s\n", cudaGetErrorString(e));
  cudaEventRecord(a);
  passB_tc_kernel<128><<<sms, TCB_THREADS, TcbCfg<128>::SMEM>>>(ws, X);
  cudaEventRecord(b);
  passB2_reduce_kernel<128><<<(2 * k * k + k + 31) / 32, PB_RED_THREADS>>>(ws, sms);
  cudaEventSynchronize(b);
  e = cudaDeviceSynchronize();
  float ms2; cudaEventElapsedTime(&ms2, a, b);
  std::vector<double> r1(2 * k * k + k), r2(2 * k * k + k);
  cudaMemcpy(r1.data(), out1, r1.size() * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(r2.data(), out2, r2.size() * 8, cudaMemcpyDeviceToHost);
  double em = 0, eg = 0, er = 0, sm = 0, sg = 0, sr = 0;
  for (int i = 0; i < k * k; ++i) { em = fmax(em, fabs(r1[i] - r2[i])); sm = fmax(sm, fabs(r1[i])); }
  for (int i = k * k; i < 2 * k * k; ++i) { eg = fmax(eg, fabs(r1[i] - r2[i])); sg = fmax(sg, fabs(r1[i])); }
  for (int i = 2 * k * k; i < 2 * k * k + k; ++i) { er = fmax(er, fabs(r1[i] - r2[i])); sr = fmax(sr, fabs(r1[i])); }
  printf("n=%lld  %s  FP64 passB2 %.3f ms | tcgen05 passB %.3f ms (%.0f GB/s of X+W)\n", (long long)n,
         cudaGetErrorString(e), ms1, ms2, 16.0 * n * k / ms2 / 1e6);
  printf("max|dM| %.3e (max|M| %.3e)  max|dG| %.3e (max|G| %.3e)  max|drr| %.3e (max|rr| %.3e)\n", em, sm, eg, sg, er, sr);
  printf("M[0..2] %.15e %.15e | %.15e %.15e\n", r1[0], r1[1], r2[0], r2[1]);
  return 0;
}
