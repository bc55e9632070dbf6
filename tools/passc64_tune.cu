// FP64 pass C tile variants at the cfg5 shape (n = 4,096,000, k = 128): CUDA-event time per launch.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/passc64_tune tools/passc64_tune.cu
#include <cstdio>
#include <cmath>
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

template <int NC, int BM, int WM, int WN>
void run(Ws ws, const double* X, double* out, int sms) {
  using CC = PassCCfg<128, NC, BM, WM, WN>;
  auto pc = passC_kernel<128, NC, BM, WM, WN>;
  if (cudaFuncSetAttribute(pc, cudaFuncAttributeMaxDynamicSharedMemorySize, CC::SMEM) != cudaSuccess) {
    printf("NC=%d BM=%d %dx%d: smem %d too large\n", NC, BM, WM, WN, CC::SMEM); cudaGetLastError(); return;
  }
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, pc, CC::THREADS, CC::SMEM);
  const int g = sms * (occ > 0 ? occ : 1);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  pc<<<dim3(g, 128 / NC), CC::THREADS, CC::SMEM>>>(ws, X, out, 1);
  cudaEventRecord(a);
  for (int r = 0; r < 3; ++r) pc<<<dim3(g, 128 / NC), CC::THREADS, CC::SMEM>>>(ws, X, out, 1);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("NC=%3d BM=%2d warps %dx%d occ %d: %.3f ms  %.1f TFLOP/s  (%s)\n", NC, BM, WM, WN, occ, ms / 3,
         2.0 * ws.n_loc * 128 * 128 / (ms / 3) / 1e9, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const int64_t n = 4096000; const int k = 128, sms = 148;
  double *X, *W, *Cs, *sc, *Xt, *ns; int* st;
  cudaMalloc(&X, n * k * 8); cudaMalloc(&W, n * k * 8); cudaMalloc(&Cs, k * k * 8); cudaMalloc(&sc, k * 8);
  cudaMalloc(&Xt, n * k * 8); cudaMalloc(&ns, 4096 * k * 8); cudaMalloc(&st, 4); cudaMemset(st, 0, 4);
  fill<<<1184, 256>>>(X, n * k, 1, 1e-3); fill<<<1184, 256>>>(W, n * k, 2, 1e-3);
  fill<<<64, 256>>>(Cs, k * k, 3, 1e-3); fill<<<1, 128>>>(sc, k, 4, 1.0);
  Ws ws{};
  ws.n_loc = n; ws.k = k; ws.kp = 128; ws.top = 0; ws.W = W; ws.Csig = Cs; ws.scal = sc; ws.status = st; ws.Xt = Xt;
  ws.nslot = ns;
  run<128, 32, 2, 8>(ws, X, Xt, sms);
  run<128, 32, 2, 4>(ws, X, Xt, sms);
  run<128, 16, 1, 8>(ws, X, Xt, sms);
  run<128, 32, 1, 8>(ws, X, Xt, sms);
  run<128, 32, 4, 4>(ws, X, Xt, sms);
  run<128, 48, 3, 4>(ws, X, Xt, sms);
  run<128, 24, 3, 4>(ws, X, Xt, sms);
  return 0;
}
