// pass-C experiment harness at the cfg5 shape (n = 4,096,000, k = 128) and cfg4 (n = 1,045,504,
// k = 32): passC tilings timed with CUDA events on random X, W, Csig.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/passc_bench tools/passc_bench.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2602_23778_b200/csrc/passes.cuh"
using namespace rf;

__global__ void fill(double* p, int64_t n, uint64_t seed) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t z = (i + 1) * 0x9E3779B97F4A7C15ull ^ seed;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull; z = (z ^ (z >> 27)) * 0x94D049BB133111EBull; z ^= z >> 31;
    p[i] = (double)(z >> 11) * 0x1p-53 - 0.5;
  }
}

template <int KP, int NC, int BM, int WM, int WN>
void run(const char* name, int64_t n, double* X, Ws ws, int sms) {
  using C = PassCCfg<KP, NC, BM, WM, WN>;
  auto kern = passC_kernel<KP, NC, BM, WM, WN>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, C::THREADS, C::SMEM);
  const int64_t ctiles = (n + BM - 1) / BM;
  const int gx = (int)std::min<int64_t>(std::max(sms * occ / (KP / NC), 1), ctiles);
  double* nslot;
  cudaMalloc(&nslot, (size_t)gx * KP * 8);
  ws.nslot = nslot;
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  kern<<<dim3(gx, KP / NC), C::THREADS, C::SMEM>>>(ws, X, 1);
  cudaEventRecord(a);
  const int reps = 3;
  for (int r = 0; r < reps; ++r) kern<<<dim3(gx, KP / NC), C::THREADS, C::SMEM>>>(ws, X, 1);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); ms /= reps;
  const double fl = 2.0 * n * KP * KP;
  printf("%s passC NC=%d BM=%d WM=%d WN=%d smem=%d occ=%d grid=%dx%d: %.3f ms  %.2f TF/s  %.0f GB/s  err=%s\n", name, NC,
         BM, WM, WN, C::SMEM, occ, gx, KP / NC, ms, fl / ms / 1e9, 24.0 * n * KP / ms / 1e6,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(nslot);
}

int main() {
  const int sms = 148;
  for (int cfg : {5, 4}) {
    const int64_t n = cfg == 5 ? 4096000 : 1045504;
    const int k = cfg == 5 ? 128 : 32;
    double *X, *W, *Xt, *Cs, *sc; int* st;
    cudaMalloc(&X, n * k * 8); cudaMalloc(&W, n * k * 8); cudaMalloc(&Xt, n * k * 8);
    cudaMalloc(&Cs, k * k * 8); cudaMalloc(&sc, k * 8); cudaMalloc(&st, 4);
    fill<<<1184, 256>>>(X, n * k, 1); fill<<<1184, 256>>>(W, n * k, 2); fill<<<64, 256>>>(Cs, k * k, 3);
    fill<<<1, 128>>>(sc, k, 4);
    cudaMemset(st, 0, 4);
    Ws ws{};
    ws.n_loc = n; ws.k = k; ws.top = 0; ws.W = W; ws.Xt = Xt; ws.Csig = Cs; ws.scal = sc; ws.status = st;
    if (cfg == 5) {
      run<128, 64, 16, 1, 8>("cfg5", n, X, ws, sms);
      run<128, 64, 32, 2, 4>("cfg5", n, X, ws, sms);
      run<128, 64, 32, 1, 8>("cfg5", n, X, ws, sms);
      run<128, 64, 64, 4, 2>("cfg5", n, X, ws, sms);
      run<128, 64, 64, 2, 4>("cfg5", n, X, ws, sms);
      run<128, 128, 32, 2, 4>("cfg5", n, X, ws, sms);
      run<128, 128, 16, 1, 8>("cfg5", n, X, ws, sms);
      run<128, 32, 32, 2, 4>("cfg5", n, X, ws, sms);
      run<128, 32, 64, 4, 2>("cfg5", n, X, ws, sms);
    } else {
      run<32, 32, 64, 4, 2>("cfg4", n, X, ws, sms);
      run<32, 32, 64, 2, 4>("cfg4", n, X, ws, sms);
      run<32, 32, 128, 4, 2>("cfg4", n, X, ws, sms);
    }
    cudaFree(X); cudaFree(W); cudaFree(Xt); cudaFree(Cs); cudaFree(sc); cudaFree(st);
  }
  return 0;
}
