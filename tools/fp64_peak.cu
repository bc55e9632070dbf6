// FP64 peak microbenchmark for B200 (sm_100a): DMMA.8x8x4 (mma.sync f64) and DFMA.
// Used once to establish the FP64 roofline denominator (MEASURED_PEAKS.json has none).
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

template<int CH>
__global__ void dmma_loop(double* out, int iters, double seed){
  double a = seed + threadIdx.x, b = seed - threadIdx.x;
  double c[CH][2];
  #pragma unroll
  for(int i=0;i<CH;i++){c[i][0]=0;c[i][1]=0;}
  for(int it=0; it<iters; ++it){
    #pragma unroll
    for(int i=0;i<CH;i++)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s=0;
  #pragma unroll
  for(int i=0;i<CH;i++) s += c[i][0]+c[i][1];
  if (s == 12345.678) out[0]=s;
}
template<int CH>
__global__ void dfma_loop(double* out, int iters, double seed){
  double a = seed + threadIdx.x*1e-9, b = 1.0 - 1e-12*threadIdx.x;
  double c[CH];
  #pragma unroll
  for(int i=0;i<CH;i++) c[i]=i;
  for(int it=0; it<iters; ++it){
    #pragma unroll
    for(int i=0;i<CH;i++) c[i] = fma(c[i], b, a);
  }
  double s=0;
  #pragma unroll
  for(int i=0;i<CH;i++) s += c[i];
  if (s == 12345.678) out[0]=s;
}
int main(){
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p,0));
  printf("device %s SMs %d clock(kHz) %d l2 %d\n", p.name, p.multiProcessorCount, p.clockRate, p.l2CacheSize);
  double* d; CK(cudaMalloc(&d, 64));
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = p.multiProcessorCount;
  for(int warps : {4, 8, 16, 32}){
    for(int blocksPerSm : {1, 2}){
      int iters = 20000;
      dim3 g(sms*blocksPerSm), b(32*warps);
      dmma_loop<8><<<g,b>>>(d, 100, 1.0); CK(cudaDeviceSynchronize());
      cudaEventRecord(e0);
      for(int r=0;r<5;r++) dmma_loop<8><<<g,b>>>(d, iters, 1.0);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms,e0,e1);
      double flops = 5.0*(double)g.x*warps*iters*8*256*2;
      printf("DMMA warps/blk %2d blk/SM %d : %.2f TFLOP/s\n", warps, blocksPerSm, flops/ms/1e9);
    }
  }
  for(int warps : {4, 8, 16, 32}){
    int iters = 20000;
    dim3 g(sms*2), b(32*warps);
    dfma_loop<8><<<g,b>>>(d, 100, 1.0); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    for(int r=0;r<5;r++) dfma_loop<8><<<g,b>>>(d, iters, 1.0);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms,e0,e1);
    double flops = 5.0*(double)g.x*b.x*iters*8*2;
    printf("DFMA warps/blk %2d blk/SM 2 : %.2f TFLOP/s\n", warps, flops/ms/1e9);
  }
  return 0;
}
