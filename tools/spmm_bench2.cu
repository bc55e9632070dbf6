// SpMM experiment harness #2: the production gather kernel (spmm_gather_kernel) against the
// previous vec kernel, an L2-hit read bandwidth probe and an HBM copy.
// cfg4 shape (2D 5-point 1024 x 1021, k = 32) and cfg5 shape (3D 7-point 160^3, k = 128).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/spmm_bench2 tools/spmm_bench2.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include "../paper_2602_23778_b200/csrc/spmm_csr.cuh"
using namespace rf;

// L2-hit bandwidth: every CTA re-reads a buffer that fits in L2 (ld.global.cg bypasses L1)
__global__ void l2_read(const double2* __restrict__ a, int64_t n2, int reps, double* out) {
  double s = 0.0;
  for (int r = 0; r < reps; ++r)
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += (int64_t)gridDim.x * blockDim.x) {
      double2 v = __ldcg(a + i);
      s += v.x + v.y;
    }
  if (s == 12345.678) out[0] = s;
}
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
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(e)); exit(1); }
  return ms / reps;
}

struct Prob {
  int64_t n, nnz; int k;
  int32_t *rp, *ci, *xoff; double *v, *X, *W, *ag; int* st;
  double bytes;
};







template <int K, int PF = 0, int LPR = 0, int MINB = 0, int UN = 8>
static void gather_case(const char* name, const Prob& p, int sms, const double* Wref, int R, int4 ord = {0, 0, 0, 0}) {
  const int occ_override = 0;
  auto kern = spmm_gather_kernel<K, false, UN, LPR, MINB>;
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 256, 0);
  if (occ_override) occ = occ_override;
  Ws ws{};
  ws.n_loc = p.n; ws.k = p.k; ws.W = p.W; ws.shift = 0.0; ws.halo = nullptr; ws.row0 = 0; ws.row1 = p.n;
  ws.ag = p.ag; ws.status = p.st;
  const int gx = sms * occ;
  cudaMemset(p.W, 0, p.n * p.k * 8);
  float ms = timeit([&] { kern<<<gx, 256>>>(ws, p.rp, p.xoff, p.v, p.X, R, p.X, ord); });
  std::vector<double> a(p.n * p.k), b(p.n * p.k);
  cudaMemcpy(a.data(), p.W, a.size() * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(b.data(), Wref, b.size() * 8, cudaMemcpyDeviceToHost);
  int64_t bad = 0;
  for (size_t i = 0; i < a.size(); ++i) bad += (a[i] != b[i]);
  printf("%s gather ord=(%d,%d,%d,%d) MINB=%d UN=%d K=%d R=%d occ=%d grid=%d: %.3f ms %6.0f GB/s  mismatches %lld\n", name, ord.x, ord.y, ord.z, ord.w, MINB, UN, K, R, occ, gx, ms,
         p.bytes / ms / 1e6, (long long)bad);
}

static Prob make(int nx, int ny, int nz, int k) {
  std::vector<int32_t> rp, ci;
  std::vector<double> v;
  build_stencil(nx, ny, nz, rp, ci, v);
  Prob p;
  p.n = (int64_t)rp.size() - 1; p.nnz = (int64_t)ci.size(); p.k = k;
  cudaMalloc(&p.rp, rp.size() * 4); cudaMalloc(&p.ci, p.nnz * 4); cudaMalloc(&p.v, p.nnz * 8);
  cudaMalloc(&p.X, p.n * k * 8); cudaMalloc(&p.W, p.n * k * 8);
  cudaMalloc(&p.ag, (size_t)148 * 64 * 128 * 4 * 8); cudaMalloc(&p.st, 4); cudaMemset(p.st, 0, 4);
  cudaMemcpy(p.rp, rp.data(), rp.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(p.ci, ci.data(), p.nnz * 4, cudaMemcpyHostToDevice);
  std::vector<int32_t> xo(p.nnz);
  for (int64_t q = 0; q < p.nnz; ++q) xo[q] = (int32_t)((int64_t)ci[q] * k / 2);
  cudaMalloc(&p.xoff, p.nnz * 4);
  cudaMemcpy(p.xoff, xo.data(), p.nnz * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(p.v, v.data(), p.nnz * 8, cudaMemcpyHostToDevice);
  std::vector<double> x(p.n * k);
  uint64_t s = 88172645463325252ull;
  for (auto& e : x) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; e = (double)(s >> 11) * 0x1p-53 - 0.5; }
  cudaMemcpy(p.X, x.data(), x.size() * 8, cudaMemcpyHostToDevice);
  p.bytes = 12.0 * p.nnz + 4.0 * (p.n + 1) + 16.0 * p.n * k;
  return p;
}

template <int VPL, int LPR>
static double* prod_case(const char* name, const Prob& p, int sms) {
  Ws ws{};
  ws.n_loc = p.n; ws.k = p.k; ws.W = p.W; ws.shift = 0.0; ws.halo = nullptr; ws.row0 = 0; ws.row1 = p.n;
  ws.ag = p.ag; ws.status = p.st;
  float ms = timeit([&] { spmm_csr_vec_kernel<VPL, LPR, false><<<sms * 8, 256>>>(ws, p.rp, p.ci, p.v, p.X, p.X); });
  printf("%s production vec kernel: %.3f ms  %.0f GB/s\n", name, ms, p.bytes / ms / 1e6);
  double* Wref;
  cudaMalloc(&Wref, p.n * p.k * 8);
  cudaMemcpy(Wref, p.W, p.n * p.k * 8, cudaMemcpyDeviceToDevice);
  return Wref;
}

int main(int argc, char** argv) {
  const int sms = 148;
  const int which = argc > 1 ? atoi(argv[1]) : 0;
  {  // L2-hit bandwidth and HBM copy
    double *buf, *out, *big, *big2;
    const int64_t n2 = (48ll << 20) / 16;
    cudaMalloc(&buf, n2 * 16); cudaMalloc(&out, 8); cudaMemset(buf, 0, n2 * 16);
    for (int g : {sms * 4, sms * 8}) {
      float ms = timeit([&] { l2_read<<<g, 512>>>((const double2*)buf, n2, 20, out); });
      printf("L2-hit read (48 MB x 20, grid %d): %.3f ms  %.0f GB/s\n", g, ms, 20.0 * n2 * 16 / ms / 1e6);
    }
    const int64_t m2 = (2ll << 30) / 16;
    cudaMalloc(&big, m2 * 16); cudaMalloc(&big2, m2 * 16);
    float mc = timeit([&] { copy_kernel<<<sms * 8, 256>>>((const double2*)big, (double2*)big2, m2); });
    printf("HBM copy 2 GiB: %.3f ms  %.0f GB/s (r+w)\n", mc, 2.0 * m2 * 16 / mc / 1e6);
    cudaFree(buf); cudaFree(big); cudaFree(big2);
  }
  if (which == 0 || which == 4) {
    Prob p = make(1024, 1021, 1, 32);
    double* Wref = prod_case<1, 16>("cfg4", p, sms);
    gather_case<32, 0, 0, 4, 5>("cfg4", p, sms, Wref, 128);
  }
  if (which == 0 || which == 5) {
    Prob p = make(160, 160, 160, 128);
    double* Wref = prod_case<2, 32>("cfg5", p, sms);
    gather_case<128, 0, 0, 2, 7>("cfg5", p, sms, Wref, 32);
    const int4 o = make_int4(5, 160, 16, 160);
    gather_case<128, 0, 0, 2, 7>("cfg5", p, sms, Wref, 32, o);
    gather_case<128, 0, 0, 3, 7>("cfg5", p, sms, Wref, 32, o);
    gather_case<128, 0, 0, 3, 4>("cfg5", p, sms, Wref, 32, o);
    gather_case<128, 0, 0, 4, 4>("cfg5", p, sms, Wref, 32, o);
    gather_case<128, 0, 0, 3, 3>("cfg5", p, sms, Wref, 32, o);
    gather_case<128, 0, 0, 2, 4>("cfg5", p, sms, Wref, 32, o);
  }
  return 0;
}
