// SpMM experiment harness at the cfg5 shape (3D 7-point stencil, 160^3, k = 128) and cfg4
// (2D 5-point, 1024 x 1021, k = 32): W = A X, variants of the gather kernel, timed with events.
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
#include "../paper_2602_23778_b200/csrc/spmm_csr.cuh"
using namespace rf;

// V1: vec kernel without the alpha/g accumulation (pure gather + store)
template <int VPL, int LPR>
__global__ void __launch_bounds__(256, 2) gather_only(int64_t n, const int32_t* __restrict__ row_ptr,
                                                     const int32_t* __restrict__ col_idx,
                                                     const double* __restrict__ val, const double* __restrict__ X,
                                                     double* __restrict__ W) {
  constexpr int RPW = 32 / LPR, K = 2 * VPL * LPR, MAXNZ = (VPL > 1) ? 4 : 8, SLOTS = 8 * RPW;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int sub = lane / LPR, l = lane % LPR, slot = warp * RPW + sub;
  for (int64_t i = (int64_t)blockIdx.x * SLOTS + slot; i < n; i += (int64_t)gridDim.x * SLOTS) {
    const int32_t p0 = row_ptr[i], p1 = row_ptr[i + 1];
    double acc[2 * VPL];
#pragma unroll
    for (int c = 0; c < 2 * VPL; ++c) acc[c] = 0.0;
    for (int32_t q0 = p0; q0 < p1; q0 += MAXNZ) {
      const int cnt = min(MAXNZ, p1 - q0);
      int32_t cols[MAXNZ];
      double vals[MAXNZ];
#pragma unroll
      for (int t = 0; t < MAXNZ; ++t)
        if (t < cnt) { cols[t] = __ldg(col_idx + q0 + t); vals[t] = __ldg(val + q0 + t); }
      double2 xs[MAXNZ][VPL];
#pragma unroll
      for (int t = 0; t < MAXNZ; ++t)
        if (t < cnt)
#pragma unroll
          for (int v = 0; v < VPL; ++v)
            xs[t][v] = __ldg(reinterpret_cast<const double2*>(X + (int64_t)cols[t] * K) + l + LPR * v);
#pragma unroll
      for (int t = 0; t < MAXNZ; ++t)
        if (t < cnt)
#pragma unroll
          for (int v = 0; v < VPL; ++v) {
            acc[2 * v] = __fma_rn(vals[t], xs[t][v].x, acc[2 * v]);
            acc[2 * v + 1] = __fma_rn(vals[t], xs[t][v].y, acc[2 * v + 1]);
          }
    }
#pragma unroll
    for (int v = 0; v < VPL; ++v)
      reinterpret_cast<double2*>(W + i * K)[l + LPR * v] = make_double2(acc[2 * v], acc[2 * v + 1]);
  }
}

// V2: pure streaming copy X -> W (HBM reference)
__global__ void copy_kernel(const double2* __restrict__ a, double2* __restrict__ b, int64_t n2) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += (int64_t)gridDim.x * blockDim.x)
    b[i] = a[i];
}

static void build_stencil(int nx, int ny, int nz, std::vector<int32_t>& rp, std::vector<int32_t>& ci,
                          std::vector<double>& v) {
  const int64_t n = (int64_t)nx * ny * nz;
  rp.assign(n + 1, 0);
  ci.clear(); v.clear();
  for (int z = 0; z < nz; ++z)
    for (int y = 0; y < ny; ++y)
      for (int x = 0; x < nx; ++x) {
        const int64_t i = x + (int64_t)nx * (y + (int64_t)ny * z);
        auto add = [&](int64_t j, double a) { ci.push_back((int32_t)j); v.push_back(a); };
        if (nz > 1 && z > 0) add(i - (int64_t)nx * ny, 1.29);
        if (y > 0) add(i - nx, 1.13);
        if (x > 0) add(i - 1, 1.0);
        add(i, 6.84);
        if (x + 1 < nx) add(i + 1, 1.0);
        if (y + 1 < ny) add(i + nx, 1.13);
        if (nz > 1 && z + 1 < nz) add(i + (int64_t)nx * ny, 1.29);
        rp[i + 1] = (int32_t)ci.size();
      }
}

template <typename F>
static float timeit(F f, int reps = 5) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  f();
  cudaDeviceSynchronize();
  cudaEventRecord(a);
  for (int r = 0; r < reps; ++r) f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms / reps;
}

template <int VPL, int LPR>
static void run_case(const char* name, int nx, int ny, int nz) {
  constexpr int K = 2 * VPL * LPR;
  std::vector<int32_t> rp, ci;
  std::vector<double> v;
  build_stencil(nx, ny, nz, rp, ci, v);
  const int64_t n = (int64_t)rp.size() - 1, nnz = (int64_t)ci.size();
  int32_t *drp, *dci; double *dv, *dX, *dW;
  cudaMalloc(&drp, rp.size() * 4); cudaMalloc(&dci, nnz * 4); cudaMalloc(&dv, nnz * 8);
  cudaMalloc(&dX, n * K * 8); cudaMalloc(&dW, n * K * 8);
  cudaMemcpy(drp, rp.data(), rp.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dci, ci.data(), nnz * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dv, v.data(), nnz * 8, cudaMemcpyHostToDevice);
  cudaMemset(dX, 0, n * K * 8);
  const double bytes = 12.0 * nnz + 4.0 * (n + 1) + 16.0 * n * K;
  const int sms = 148;
  for (int g : {sms * 2, sms * 4, sms * 8, sms * 16}) {
    float ms = timeit([&] { gather_only<VPL, LPR><<<g, 256>>>(n, drp, dci, dv, dX, dW); });
    printf("%s gather_only grid %5d: %.3f ms  %.0f GB/s (alg bytes)\n", name, g, ms, bytes / ms / 1e6);
  }
  // full kernel (with dd alpha/g) through a Ws
  Ws ws{};
  ws.n_loc = n; ws.k = K; ws.W = dW; ws.shift = 0.0; ws.halo = nullptr; ws.row0 = 0; ws.row1 = n;
  double* ag; int* st;
  cudaMalloc(&ag, (size_t)sms * 8 * K * 4 * 8); cudaMalloc(&st, 4); cudaMemset(st, 0, 4);
  ws.ag = ag; ws.status = st;
  float ms = timeit([&] { spmm_csr_vec_kernel<VPL, LPR, false><<<sms * 8, 256>>>(ws, drp, dci, dv, dX, dX); });
  printf("%s full vec kernel (dd alpha/g): %.3f ms  %.0f GB/s\n", name, ms, bytes / ms / 1e6);
  float mc = timeit([&] { copy_kernel<<<sms * 8, 256>>>((const double2*)dX, (double2*)dW, n * K / 2); });
  printf("%s copy X->W: %.3f ms  %.0f GB/s\n", name, mc, 16.0 * n * K / mc / 1e6);
  cudaFree(drp); cudaFree(dci); cudaFree(dv); cudaFree(dX); cudaFree(dW); cudaFree(ag); cudaFree(st);
}

int main() {
  run_case<1, 16>("cfg4", 1024, 1021, 1);
  run_case<2, 32>("cfg5", 160, 160, 160);
  return 0;
}
