// spmm_csr.cuh -- S1 for CSR A: W = A X^ - shift X^ (Alg. 4 line 1; Sec. 5.1,
// PAPER.md:1203) fused with the S2 partials alpha_j and g_j (lines 3-4).
//
// One warp per row; lanes across the k columns (lane l owns columns l, l+32, ...), so the
// gathered row X^[col] is read as one coalesced 256-byte segment per 32 columns.  The
// row's (col, val) pairs are loaded once per warp (lane t holds nonzero t of the chunk)
// and broadcast with shuffles.  Each output is an fma chain in ascending CSR order --
// the same chain as the oracle, so W is bit-identical given identical X^ (P3).
// Rows are dealt block-cyclically so the whole grid advances through A together and the gathered
// rows hit L2: at cfg5 the +-z neighbours are 25,600 rows (26 MB) apart.
#pragma once
#include "common.cuh"

namespace rf {

template <int CPL, bool HALO>   // columns per lane = ceil(k / 32); HALO: row-partitioned X
__global__ void __launch_bounds__(256) spmm_csr_kernel(Ws ws, const int32_t* __restrict__ row_ptr,
                                                       const int32_t* __restrict__ col_idx,
                                                       const double* __restrict__ val,
                                                       const double* __restrict__ X,      // unused (see xrow)
                                                       const double* __restrict__ Xloc) {  // local rows
  __shared__ dd sa[8][KMAX], sg[8][KMAX];
  if (*ws.status != ST_OK) return;
  const int k = ws.k;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  dd a[CPL], g[CPL];
#pragma unroll
  for (int c = 0; c < CPL; ++c) a[c] = g[c] = dd{0.0, 0.0};
  // block-cyclic rows: all CTAs sweep the matrix together, so the rows a stencil gathers
  // (+-1 grid line / plane) were touched recently and are still in L2
  for (int64_t i = (int64_t)blockIdx.x * 8 + warp; i < ws.n_loc; i += (int64_t)gridDim.x * 8) {
    const int32_t p0 = row_ptr[i], p1 = row_ptr[i + 1];   // absolute offsets into col_idx / val
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
        const double* xr = HALO ? xrow(ws, Xloc, col, k) : Xloc + (int64_t)col * k;
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

// Vectorised variant for even k = 2 VPL LPR: a row is handled by LPR lanes, each owning VPL
// double2 column pairs (LPR = 32 / rows-per-warp), so small k still issues full 256-byte
// warp transactions.  Up to MAXNZ gathers of a row are issued before the (in-order) fma chain
// consumes them, which keeps ~MAXNZ x 256 bytes in flight per row.
template <int VPL, int LPR, bool HALO>
__global__ void __launch_bounds__(256, 2) spmm_csr_vec_kernel(Ws ws, const int32_t* __restrict__ row_ptr,
                                                           const int32_t* __restrict__ col_idx,
                                                           const double* __restrict__ val,
                                                           const double* __restrict__ X,
                                                           const double* __restrict__ Xloc) {
  constexpr int RPW = 32 / LPR, K = 2 * VPL * LPR, MAXNZ = (VPL > 1) ? 4 : 8, SLOTS = 8 * RPW;
  __shared__ dd sa[SLOTS][K], sg[SLOTS][K];
  if (*ws.status != ST_OK) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int sub = lane / LPR, l = lane % LPR, slot = warp * RPW + sub;
  // alpha / g: plain FP64 fma sums over blocks of ABLK rows, merged into double-double
  // accumulators (relative error <= ABLK u for the same-sign terms of x^2 and x w, against
  // ~u^2 for a full double-double chain at a quarter of its FP64 instructions)
  constexpr int ABLK = 8;
  dd a[2 * VPL], g[2 * VPL];
  double ba[2 * VPL], bg[2 * VPL];
#pragma unroll
  for (int c = 0; c < 2 * VPL; ++c) { a[c] = g[c] = dd{0.0, 0.0}; ba[c] = bg[c] = 0.0; }
  int nb = 0;
  for (int64_t i = (int64_t)blockIdx.x * SLOTS + slot; i < ws.n_loc; i += (int64_t)gridDim.x * SLOTS) {
    const int32_t p0 = row_ptr[i], p1 = row_ptr[i + 1];   // absolute offsets into col_idx / val
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
            xs[t][v] = __ldg(reinterpret_cast<const double2*>(HALO ? xrow(ws, Xloc, cols[t], K)
                                                                   : Xloc + (int64_t)cols[t] * K) + l + LPR * v);
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
    for (int v = 0; v < VPL; ++v) {
      const double2 x = reinterpret_cast<const double2*>(Xloc + i * K)[l + LPR * v];
      double w0 = acc[2 * v], w1 = acc[2 * v + 1];
      if (ws.shift != 0.0) { w0 = __fma_rn(-ws.shift, x.x, w0); w1 = __fma_rn(-ws.shift, x.y, w1); }
      reinterpret_cast<double2*>(ws.W + i * K)[l + LPR * v] = make_double2(w0, w1);
      ba[2 * v] = __fma_rn(x.x, x.x, ba[2 * v]);
      ba[2 * v + 1] = __fma_rn(x.y, x.y, ba[2 * v + 1]);
      bg[2 * v] = __fma_rn(x.x, w0, bg[2 * v]);
      bg[2 * v + 1] = __fma_rn(x.y, w1, bg[2 * v + 1]);
    }
    if (++nb == ABLK) {
      nb = 0;
#pragma unroll
      for (int c = 0; c < 2 * VPL; ++c) {
        dd_add1(a[c], ba[c]); dd_add1(g[c], bg[c]);
        ba[c] = bg[c] = 0.0;
      }
    }
  }
#pragma unroll
  for (int c = 0; c < 2 * VPL; ++c) { dd_add1(a[c], ba[c]); dd_add1(g[c], bg[c]); }
#pragma unroll
  for (int v = 0; v < VPL; ++v) {
    const int j = 2 * (l + LPR * v);
    sa[slot][j] = a[2 * v]; sa[slot][j + 1] = a[2 * v + 1];
    sg[slot][j] = g[2 * v]; sg[slot][j + 1] = g[2 * v + 1];
  }
  __syncthreads();
  for (int j = threadIdx.x; j < K; j += 256) {
    dd ta = sa[0][j], tg = sg[0][j];
    for (int q = 1; q < SLOTS; ++q) { dd_add(ta, sa[q][j]); dd_add(tg, sg[q][j]); }
    double* sl = ws.ag + ((int64_t)blockIdx.x * K + j) * 4;
    sl[0] = ta.hi; sl[1] = ta.lo; sl[2] = tg.hi; sl[3] = tg.lo;
  }
}

}  // namespace rf
