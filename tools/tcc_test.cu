// pass C on tcgen05 (mixed precision) vs the FP64 DMMA pass C: accuracy of X~ and of the column
// sums of squares, and timing.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/tcc_test tools/tcc_test.cu
#include <cstdio>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
#include "../paper_2602_23778_b200/csrc/passes.cuh"
#include "../paper_2602_23778_b200/csrc/tc_passes.cuh"
#include "../paper_2602_23778_b200/csrc/ozaki.cuh"
using namespace rf;

__global__ void fill(double* p, int64_t n, uint64_t seed, double scale, double off) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t z = (i + 1) * 0x9E3779B97F4A7C15ull ^ seed;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull; z = (z ^ (z >> 27)) * 0x94D049BB133111EBull; z ^= z >> 31;
    p[i] = ((double)(z >> 11) * 0x1p-53 - 0.5) * scale + off;
  }
}

int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? atoll(argv[1]) : 4096000;
  const int top = argc > 2 ? atoi(argv[2]) : 128;
  const int k = 128, sms = 148;
  double *X, *W, *Cs, *sc, *Xt1, *Xt2, *ns1, *ns2; int* st;
  cudaMalloc(&X, n * k * 8); cudaMalloc(&W, n * k * 8); cudaMalloc(&Cs, k * k * 8); cudaMalloc(&sc, k * 8);
  cudaMalloc(&Xt1, n * k * 8); cudaMalloc(&Xt2, n * k * 8); cudaMalloc(&st, 4);
  cudaMalloc(&ns1, 4096 * k * 8); cudaMalloc(&ns2, 4096 * k * 8);
  fill<<<1184, 256>>>(X, n * k, 1, 1.0 / sqrt((double)n), 0.0);
  fill<<<1184, 256>>>(W, n * k, 2, 1.0 / sqrt((double)n), 0.0);
  fill<<<64, 256>>>(Cs, k * k, 3, 1e-3, 0.0);     // O(residual) correction coefficients
  fill<<<1, 128>>>(sc, k, 4, 1.0, 1.0);
  cudaMemset(st, 0, 4);
  cudaMemset(Xt1, 0, n * k * 8); cudaMemset(Xt2, 0, n * k * 8);
  Ws ws{};
  ws.n_loc = n; ws.k = k; ws.kp = 128; ws.top = top; ws.W = W; ws.Csig = Cs; ws.scal = sc; ws.status = st;
  using CC = PassCCfg<128, 128, 32, 2, 8>;
  auto pc = passC_kernel<128, 128, 32, 2, 8>;
  cudaFuncSetAttribute(pc, cudaFuncAttributeMaxDynamicSharedMemorySize, CC::SMEM);
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, pc, CC::THREADS, CC::SMEM);
  const int g1 = sms * occ;
  ws.Xt = Xt1; ws.nslot = ns1;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  pc<<<dim3(g1, 1), CC::THREADS, CC::SMEM>>>(ws, X, Xt1, 1);
  cudaEventRecord(a);
  pc<<<dim3(g1, 1), CC::THREADS, CC::SMEM>>>(ws, X, Xt1, 1);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms1; cudaEventElapsedTime(&ms1, a, b);
  cudaFuncSetAttribute(passC_tc_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, TccCfg<128>::SMEM);
  ws.Xt = Xt2; ws.nslot = ns2;
  passC_tc_kernel<128><<<sms, TCC_THREADS, TccCfg<128>::SMEM>>>(ws, X, Xt2);
  cudaError_t e = cudaDeviceSynchronize();
  printf("first tc launch: %s\n", cudaGetErrorString(e));
  cudaEventRecord(a);
  passC_tc_kernel<128><<<sms, TCC_THREADS, TccCfg<128>::SMEM>>>(ws, X, Xt2);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  e = cudaDeviceSynchronize();
  float ms2; cudaEventElapsedTime(&ms2, a, b);
  // pass C on the INT8 tensor cores (FP64 accuracy)
  double *Xt3, *ns3;
  cudaMalloc(&Xt3, n * k * 8); cudaMalloc(&ns3, 4096 * k * 8); cudaMemset(Xt3, 0, n * k * 8);
  cudaFuncSetAttribute(passC_oz_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, OZC_SMEM);
  ws.Xt = Xt3; ws.nslot = ns3;
  passC_oz_kernel<<<sms, OZC_THREADS, OZC_SMEM>>>(ws, X, Xt3);
  cudaError_t e3 = cudaDeviceSynchronize();
  cudaEventRecord(a);
  passC_oz_kernel<<<sms, OZC_THREADS, OZC_SMEM>>>(ws, X, Xt3);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms3; cudaEventElapsedTime(&ms3, a, b);
  std::vector<double> h3(n * k);
  cudaMemcpy(h3.data(), Xt3, n * k * 8, cudaMemcpyDeviceToHost);
  std::vector<double> h1(n * k), h2(n * k), hx(n * k), hw(n * k), n1(g1 * k), n2(sms * k), hc(k * k), hs(k);
  cudaMemcpy(h1.data(), Xt1, n * k * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(h2.data(), Xt2, n * k * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(n1.data(), ns1, g1 * k * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(n2.data(), ns2, sms * k * 8, cudaMemcpyDeviceToHost);
  double ex = 0, sx = 0, en = 0, sn = 0;
  for (int64_t i = top * k; i < n * k; ++i) { ex = fmax(ex, fabs(h1[i] - h2[i])); sx = fmax(sx, fabs(h1[i])); }
  int untouched = 1;
  for (int64_t i = 0; i < top * k; ++i) untouched &= (h2[i] == 0.0);
  for (int j = 0; j < k; ++j) {
    double s1 = 0, s2 = 0;
    for (int c = 0; c < g1; ++c) s1 += n1[c * k + j];
    for (int c = 0; c < sms; ++c) s2 += n2[c * k + j];
    en = fmax(en, fabs(s1 - s2) / s1);
  }
  // size of the correction term x Csig (sampled rows)
  cudaMemcpy(hx.data(), X, n * k * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(hc.data(), Cs, k * k * 8, cudaMemcpyDeviceToHost);
  for (int64_t i = top; i < n; i += 997)
    for (int j = 0; j < k; ++j) {
      double s = 0;
      for (int l = 0; l < k; ++l) s += hx[i * k + l] * hc[l * k + j];
      sn = fmax(sn, fabs(s));
    }
  printf("n=%lld top=%d  %s  FP64 passC %.3f ms | tcgen05 passC %.3f ms (%.0f GB/s of X+W+X~)\n", (long long)n, top,
         cudaGetErrorString(e), ms1, ms2, 24.0 * (n - top) * k / ms2 / 1e6);
  printf("max|dX~| %.3e (max|X~| %.3e, max|X Csig| ~%.3e)  max rel d(norm^2) %.3e  top rows untouched %d\n", ex, sx, sn,
         en, untouched);
  double e3x = 0;
  for (int64_t i = top * k; i < n * k; ++i) e3x = fmax(e3x, fabs(h1[i] - h3[i]));
  printf("INT8 (ozaki) passC %.3f ms (%.0f GB/s, %s): max|dX~| vs FP64 %.3e\n", ms3, 24.0 * (n - top) * k / ms3 / 1e6,
         cudaGetErrorString(e3), e3x);
  return 0;
}
