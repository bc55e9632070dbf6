// spmm_csr.cuh -- S1 for CSR A: W = A X^ - shift X^ (Alg. 4 line 1; Sec. 5.1,
// PAPER.md:1203) fused with the S2 partials alpha_j and g_j (lines 3-4).
//
// One warp per row; lanes across the k columns (lane l owns columns l, l+32, ...), so the
// gathered row X^[col] is read as one coalesced 256-byte segment per 32 columns.  The
// row's (col, val) pairs are loaded once per warp (lane t holds nonzero t of the chunk)
// and broadcast with shuffles.  Each output is an fma chain in ascending CSR order --
// the same chain as the oracle, so W is bit-identical given identical X^ (P3).
// The gathered rows hit L2: at cfg5 the +-z neighbours are 25,600 rows (26 MB) apart.
#pragma once
#include "common.cuh"

namespace rf {

template <int CPL>   // columns per lane = ceil(k / 32)
__global__ void __launch_bounds__(256) spmm_csr_kernel(Ws ws, const int32_t* __restrict__ row_ptr,
                                                       const int32_t* __restrict__ col_idx,
                                                       const double* __restrict__ val,
                                                       const double* __restrict__ X,   // gathered (global rows)
                                                       const double* __restrict__ Xloc) {  // local rows
  __shared__ dd sa[8][KMAX], sg[8][KMAX];
  if (*ws.status != ST_OK) return;
  const int k = ws.k;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t rows_per = (ws.n_loc + gridDim.x - 1) / gridDim.x;
  const int64_t rb = (int64_t)blockIdx.x * rows_per;
  const int64_t re = (rb + rows_per < ws.n_loc) ? rb + rows_per : ws.n_loc;
  const int32_t base = row_ptr[0];
  dd a[CPL], g[CPL];
#pragma unroll
  for (int c = 0; c < CPL; ++c) a[c] = g[c] = dd{0.0, 0.0};

  for (int64_t i = rb + warp; i < re; i += 8) {
    const int32_t p0 = row_ptr[i] - base, p1 = row_ptr[i + 1] - base;
    double acc[CPL];
#pragma unroll
    for (int c = 0; c < CPL; ++c) acc[c] = 0.0;
    for (int32_t q0 = p0; q0 < p1; q0 += 32) {
      const int cnt = min(32, p1 - q0);
      int32_t mycol = 0;
      double myval = 0.0;
      if (lane < cnt) { mycol = col_idx[q0 + lane]; myval = val[q0 + lane]; }
      for (int t = 0; t < cnt; ++t) {
        const int32_t col = __shfl_sync(0xffffffffu, mycol, t);
        const double v = __shfl_sync(0xffffffffu, myval, t);
        const double* xr = X + (int64_t)col * k;
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
          const int j = lane + 32 * c;
          if (j < k) acc[c] = __fma_rn(v, __ldg(xr + j), acc[c]);
        }
      }
    }
    const double* xi = Xloc + i * k;
    double* wi = ws.W + i * k;
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      const int j = lane + 32 * c;
      if (j < k) {
        const double x = xi[j];
        double w = acc[c];
        if (ws.shift != 0.0) w = __fma_rn(-ws.shift, x, w);
        wi[j] = w;
        dd_add_prod(a[c], x, x);
        dd_add_prod(g[c], x, w);
      }
    }
  }
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    const int j = lane + 32 * c;
    if (j < k) { sa[warp][j] = a[c]; sg[warp][j] = g[c]; }
  }
  __syncthreads();
  for (int j = threadIdx.x; j < k; j += 256) {
    dd ta = sa[0][j], tg = sg[0][j];
    for (int w = 1; w < 8; ++w) { dd_add(ta, sa[w][j]); dd_add(tg, sg[w][j]); }
    double* slot = ws.ag + ((int64_t)blockIdx.x * k + j) * 4;
    slot[0] = ta.hi; slot[1] = ta.lo; slot[2] = tg.hi; slot[3] = tg.lo;
  }
}

}  // namespace rf
