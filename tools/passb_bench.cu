// pass-B experiment harness at the cfg5 shape (n = 4,096,000, k = 128) and cfg4 (n = 1,045,504,
// k = 32): passB2 variants (warp tiling, rows per stage) timed with CUDA events on random X, W.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/passb_bench tools/passb_bench.cu
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
#include "../paper_2602_23778_b200/csrc/passes.cuh"
using namespace rf;

template <int KP, int WA_, int WB_, int BR_, int MODE>
__global__ void __launch_bounds__(PassB2Cfg<KP, WA_, WB_, BR_>::THREADS)
exp_kernel(Ws ws, const double* __restrict__ X, int vec16) {
  using C = PassB2Cfg<KP, WA_, WB_, BR_>;
  constexpr int THREADS = C::THREADS, BR = C::BR, TB = C::TB;
  extern __shared__ __align__(16) double smem[];
  __shared__ double sd[KP];
  __shared__ double srr[2][THREADS];
  if (*ws.status != ST_OK) return;
  const int k = ws.k, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wa = warp / C::WB, wb = warp % C::WB;
  const int tb = blockIdx.x, b0 = tb * TB;                    // [R | X] columns [b0, b0 + 64)
  const int rw = (MODE == 1) ? 0 : ((b0 < KP) ? min(TB, KP - b0) : 0);
  const int64_t rows = ws.n_loc - ws.top;
  const int64_t per = ((rows + gridDim.y - 1) / gridDim.y + BR - 1) / BR * BR;
  const int64_t rb = ws.top + (int64_t)blockIdx.y * per;
  const int64_t re = (rb + per < ws.n_loc) ? rb + per : ws.n_loc;
  const int nit = (re > rb) ? (int)((re - rb + BR - 1) / BR) : 0;
  for (int j = tid; j < KP; j += THREADS) sd[j] = (j < k) ? ws.d[j] : 0.0;
  double* Xs = smem;
  double* Wsm = smem + 2 * C::XST;
  // this warp's MMAs: skipped when its block lies strictly below the diagonal of G = X^T X
  const int a_lo = wa * C::WTA, bw = b0 + wb * C::WTB;       // first a row, first [R|X] column
  const bool active = !(bw >= KP && a_lo >= (bw - KP) + C::WTB);
  // R chunks: the thread that copies W[r][b0+c..] also copies X[r][b0+c..], so it can form those
  // R entries as soon as its own copies land (no barrier).  Its R columns are fixed.
  const int rpair = vec16 ? 2 : 1;
  const int rcpr = (rw > 0) ? rw / rpair : 1;                 // R chunks per row
  const int rcol = (tid % rcpr) * rpair;                      // this thread's R column(s) b0 + rcol (+1)

  auto load = [&](int buf, int it) {
    const int64_t r0 = rb + (int64_t)it * BR;
    double* xs = Xs + buf * C::XST;
    double* wsb = Wsm + buf * C::WST;
    if (vec16) {
      for (int c = tid; c < BR * rw / 2; c += THREADS) {     // paired W / X chunks of the R columns
        const int r = c / (rw / 2), cc = (c % (rw / 2)) * 2;
        const int64_t g = r0 + r;
        const bool ok = (g < re) && (b0 + cc < k);
        if (MODE != 7) cp_async16(wsb + r * C::LDW + cc, ws.W + (ok ? g * k + b0 + cc : 0), ok);
        cp_async16(xs + r * C::LDX + b0 + cc, X + (ok ? g * k + b0 + cc : 0), ok);
      }
      constexpr int H = KP / 2;
      for (int c = tid; c < BR * H; c += THREADS) {           // the other X columns
        const int r = c / H, cc = (c % H) * 2;
        if (cc >= b0 && cc < b0 + rw) continue;
        const int64_t g = r0 + r;
        const bool ok = (g < re) && (cc < k);
        cp_async16(xs + r * C::LDX + cc, X + (ok ? g * k + cc : 0), ok);
      }
    } else {
      for (int c = tid; c < BR * rw; c += THREADS) {
        const int r = c / rw, cc = c % rw;
        const int64_t g = r0 + r;
        const bool ok = (g < re) && (b0 + cc < k);
        cp_async8(wsb + r * C::LDW + cc, ws.W + (ok ? g * k + b0 + cc : 0), ok);
        cp_async8(xs + r * C::LDX + b0 + cc, X + (ok ? g * k + b0 + cc : 0), ok);
      }
      for (int c = tid; c < BR * KP; c += THREADS) {
        const int r = c / KP, cc = c % KP;
        if (cc >= b0 && cc < b0 + rw) continue;
        const int64_t g = r0 + r;
        const bool ok = (g < re) && (cc < k);
        cp_async8(xs + r * C::LDX + cc, X + (ok ? g * k + cc : 0), ok);
      }
    }
  };
  double rr0 = 0.0, rr1 = 0.0;
  // R = W - X D for this thread's own (landed) chunks of stage buffer buf, in place (fma as in the oracle)
  auto form_r = [&](int buf) {
    const double* xs = Xs + buf * C::XST;
    double* wsb = Wsm + buf * C::WST;
    const double d0 = sd[b0 + rcol], d1 = sd[b0 + rcol + (rpair - 1)];
    for (int c = tid; c < BR * rcpr; c += THREADS) {
      const int r = c / rcpr;
      const double v0 = __fma_rn(-xs[r * C::LDX + b0 + rcol], d0, wsb[r * C::LDW + rcol]);
      wsb[r * C::LDW + rcol] = v0;
      if (MODE != 5) rr0 = __fma_rn(v0, v0, rr0);
      if (rpair == 2) {
        const double v1 = __fma_rn(-xs[r * C::LDX + b0 + rcol + 1], d1, wsb[r * C::LDW + rcol + 1]);
        wsb[r * C::LDW + rcol + 1] = v1;
        if (MODE != 5) rr1 = __fma_rn(v1, v1, rr1);
      }
    }
  };

  double acc[C::MI][C::NI][2];
#pragma unroll
  for (int i = 0; i < C::MI; ++i)
#pragma unroll
    for (int j = 0; j < C::NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  if (nit > 0) load(0, 0);
  cp_async_commit();
  __syncthreads();                                            // sd visible to form_r
  cp_async_wait<0>();
  if (rw > 0 && nit > 0) form_r(0);
  // iteration it: [barrier] issue stage it+1 -> MMAs of stage it -> wait own copies of it+1 -> R(it+1)
  for (int it = 0; it < nit; ++it) {
    const int cur = it & 1;
    __syncthreads();
    if (MODE != 2 && MODE != 3 && it + 1 < nit) load(cur ^ 1, it + 1);
    cp_async_commit();
    const double* xs = Xs + cur * C::XST;
    const double* wsb = Wsm + cur * C::WST;
    if (MODE == 4 && rw > 0) {
      cp_async_wait<1>();
      __syncthreads();
      if (it > 0) form_r(cur);
      __syncthreads();
    }
    if (active) {
#pragma unroll
      for (int kk = 0; kk < BR; kk += 4) {
        const int row = kk + (lane & 3);
        double a[C::MI], b[C::NI];
#pragma unroll
        for (int i = 0; i < C::MI; ++i) a[i] = (MODE == 3) ? (double)(i + kk) : xs[row * C::LDX + a_lo + i * 8 + (lane >> 2)];
#pragma unroll
        for (int j = 0; j < C::NI; ++j) {
          const int cb8 = bw + j * 8;                         // 8-column block: all R or all X (warp-uniform)
          b[j] = (MODE == 3) ? (double)(j - kk) : (cb8 < KP) ? wsb[row * C::LDW + (cb8 - b0) + (lane >> 2)] : xs[row * C::LDX + cb8 - KP + (lane >> 2)];
        }
#pragma unroll
        for (int i = 0; i < C::MI; ++i)
#pragma unroll
          for (int j = 0; j < C::NI; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
      }
    }
    cp_async_wait<0>();
    if (MODE != 4 && MODE != 6 && rw > 0 && it + 1 < nit) form_r(cur ^ 1);
  }
  if (active) {
    double* out = ws.bpart + ((int64_t)blockIdx.y * C::NT + tb) * (C::TA * TB);
#pragma unroll
    for (int i = 0; i < C::MI; ++i)
#pragma unroll
      for (int j = 0; j < C::NI; ++j) {
        const int ra = a_lo + i * 8 + (lane >> 2);
        const int cb = wb * C::WTB + j * 8 + 2 * (lane & 3);
        out[ra * TB + cb] = acc[i][j][0];
        out[ra * TB + cb + 1] = acc[i][j][1];
      }
  }
  if (rw > 0) {   // threads t, t + rcpr, ... share the R column(s) b0 + rcol (+1): fixed-order sum
    srr[0][tid] = rr0;
    srr[1][tid] = rr1;
    __syncthreads();
    if (tid < rcpr) {
      double s0 = srr[0][tid], s1 = srr[1][tid];
      for (int q = 1; q < THREADS / rcpr; ++q) { s0 += srr[0][q * rcpr + tid]; s1 += srr[1][q * rcpr + tid]; }
      ws.brr[(int64_t)blockIdx.y * KP + b0 + rcol] = s0;
      if (rpair == 2) ws.brr[(int64_t)blockIdx.y * KP + b0 + rcol + 1] = s1;
    }
  }
}


__global__ void fill(double* p, int64_t n, uint64_t seed) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t z = (i + 1) * 0x9E3779B97F4A7C15ull ^ seed;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull; z = (z ^ (z >> 27)) * 0x94D049BB133111EBull; z ^= z >> 31;
    p[i] = (double)(z >> 11) * 0x1p-53 - 0.5;
  }
}

template <int KP, int WA, int WB, int BR, int MODE = 0>
void run(const char* name, int64_t n, double* X, double* W, Ws ws, int sms) {
  using C = PassB2Cfg<KP, WA, WB, BR>;
  auto kern = MODE ? exp_kernel<KP, WA, WB, BR, MODE> : passB2_kernel<KP, WA, WB, BR>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, C::THREADS, C::SMEM);
  constexpr bool PR = C::PAIRED && MODE == 0;
  const int gy = PR ? 2 * (sms * occ / 7) : sms * occ / C::NT;
  double* bpart; double* brr;
  cudaMalloc(&bpart, (size_t)gy * C::NT * C::TA * C::TB * 8);
  cudaMalloc(&brr, (size_t)gy * KP * 8);
  ws.bpart = bpart; ws.brr = brr; ws.n_chunk = gy;
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  const dim3 grid = PR ? dim3(7 * (gy / 2)) : dim3(C::NT, gy);
  kern<<<grid, C::THREADS, C::SMEM>>>(ws, X, 1);
  cudaEventRecord(a);
  const int reps = 3;
  for (int r = 0; r < reps; ++r) kern<<<grid, C::THREADS, C::SMEM>>>(ws, X, 1);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); ms /= reps;
  const double mac = (double)n * (KP * KP + KP * KP - (KP > 64 ? 64.0 * 64.0 : 0.0));
  printf("%s mode %d passB2 WA=%d WB=%d BR=%d smem=%d occ=%d grid=%dx%d: %.3f ms  %.2f TF/s (MMA flops)  err=%s\n", name, MODE, WA, WB,
         BR, C::SMEM, occ, C::NT, gy, ms, 2 * mac / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
  cudaFree(bpart); cudaFree(brr);
}

int main() {
  const int sms = 148;
  for (int cfg : {5, 4}) {
    const int64_t n = cfg == 5 ? 4096000 : 1045504;
    const int k = cfg == 5 ? 128 : 32;
    double *X, *W, *d; int* st;
    cudaMalloc(&X, n * k * 8); cudaMalloc(&W, n * k * 8); cudaMalloc(&d, k * 8); cudaMalloc(&st, 4);
    fill<<<1184, 256>>>(X, n * k, 1); fill<<<1184, 256>>>(W, n * k, 2); fill<<<1, 128>>>(d, k, 3);
    cudaMemset(st, 0, 4);
    Ws ws{};
    ws.n_loc = n; ws.k = k; ws.top = 0; ws.W = W; ws.d = d; ws.status = st;
    if (cfg == 5) {
      run<128, 2, 4, 32>("cfg5", n, X, W, ws, sms);
      run<128, 2, 4, 32, 1>("cfg5", n, X, W, ws, sms);
      run<128, 2, 4, 32, 2>("cfg5", n, X, W, ws, sms);
      run<128, 2, 4, 32, 3>("cfg5", n, X, W, ws, sms);
      run<128, 4, 4, 32>("cfg5", n, X, W, ws, sms);
    } else {
      run<32, 2, 4, 32>("cfg4", n, X, W, ws, sms);
      run<32, 2, 4, 64>("cfg4", n, X, W, ws, sms);
      run<32, 2, 4, 128>("cfg4", n, X, W, ws, sms);
      run<32, 1, 8, 64>("cfg4", n, X, W, ws, sms);
      run<32, 2, 4, 32, 1>("cfg4", n, X, W, ws, sms);
      run<32, 2, 4, 32, 2>("cfg4", n, X, W, ws, sms);
      run<32, 2, 4, 32, 3>("cfg4", n, X, W, ws, sms);
    }
    cudaFree(X); cudaFree(W); cudaFree(d); cudaFree(st);
  }
  return 0;
}
