// Latency of dependent FP64 operations on one thread (clock64): DFMA, DADD, DMUL, DDIV, DSQRT,
// and of a dependent shared-memory load chain -- the numbers behind the k x k chain's design.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_latency tools/fp64_latency.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat(double* out, long long* cyc, double a, double b, int n) {
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, b, a);
  long long t1 = clock64();
  double y = a;
  for (int i = 0; i < n; ++i) y = y + b;
  long long t2 = clock64();
  double z = a;
  for (int i = 0; i < n; ++i) z = z / b;
  long long t3 = clock64();
  double w = a;
  for (int i = 0; i < n; ++i) w = sqrt(w + b);
  long long t4 = clock64();
  __shared__ int idx[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) idx[i] = (i * 7 + 1) & 1023;
  __syncthreads();
  int p = 0;
  long long t5 = clock64();
  for (int i = 0; i < n; ++i) p = idx[p];
  long long t6 = clock64();
  float f = (float)a;
  for (int i = 0; i < n; ++i) f = fmaf(f, (float)b, (float)a);
  long long t7 = clock64();
  out[0] = x + y + z + w + p + f;
  cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t6 - t5; cyc[5] = t7 - t6;
}

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
// one warp: a dependent DMMA chain, then 8 independent chains
__global__ void dmma_lat(double* out, long long* cyc, double a, double b, int n) {
  double c0 = 0, c1 = 0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) dmma(c0, c1, a, b);
  long long t1 = clock64();
  double d[8][2] = {};
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int u = 0; u < 8; ++u) dmma(d[u][0], d[u][1], a, b);
  long long t2 = clock64();
  double s = c0 + c1;
  for (int u = 0; u < 8; ++u) s += d[u][0] + d[u][1];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; }
}

int main() {
  double* o; long long* c;
  cudaMalloc(&o, 8); cudaMalloc(&c, 64);
  const int n = 4096;
  lat<<<1, 32>>>(o, c, 0.999, 1.0000001, n);
  lat<<<1, 32>>>(o, c, 0.999, 1.0000001, n);
  long long h[6];
  cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
  const char* nm[6] = {"DFMA", "DADD", "DDIV", "DSQRT+DADD", "LDS (dependent)", "FFMA"};
  for (int i = 0; i < 6; ++i) printf("%-18s %.1f cycles per dependent op\n", nm[i], (double)h[i] / n);
  double* o2; cudaMalloc(&o2, 32 * 8);
  dmma_lat<<<1, 32>>>(o2, c, 1.0, 1e-9, 1024);
  dmma_lat<<<1, 32>>>(o2, c, 1.0, 1e-9, 1024);
  cudaMemcpy(h, c, 2 * sizeof(long long), cudaMemcpyDeviceToHost);
  printf("DMMA m8n8k4 dependent: %.1f cycles; 8 independent chains: %.1f cycles per DMMA (one warp)\n",
         (double)h[0] / 1024, (double)h[1] / (8.0 * 1024));
  return 0;
}
