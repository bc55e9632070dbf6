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
                                                       const double* __restrict__ X,      // own rows (x_i)
                                                       const double* __restrict__ Xloc) {  // gathered rows
  __shared__ dd sa[8][KMAX], sg[8][KMAX];
  griddep_wait();   // (programmatic dependent launch: the predecessor's writes are visible after this)
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
    const double* xi = X + i * k;
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
  griddep_wait();   // (programmatic dependent launch: the predecessor's writes are visible after this)
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
      const double2 x = reinterpret_cast<const double2*>(X + i * K)[l + LPR * v];   // own row
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


// ---------------------------------------------------------------- spmm_gather (production CSR S1)
// For k in {2, 4, ..., 128}.  The vec kernel above is latency bound: each row is a chain of three
// dependent global round trips (row_ptr -> col/val -> the gathered X rows) with ~16 rows in flight
// per SM (cfg5: 1.9 TB/s).  Here
//   * work item = a chunk of R consecutive rows; chunks are dealt block-cyclically over the
//     persistent grid, so the whole grid sweeps A together: the X rows a banded matrix gathers
//     again (the +-y / +-z stencil neighbours) are still in L2, and consecutive rows of a chunk,
//     processed side by side by the CTA's row groups, share their x-neighbour rows through L1;
//   * the chunk's row_ptr and (gather offset, val) are staged in shared memory by cp.async two
//     and one chunks ahead, so only the X gathers are left on a row's critical path (R <= RMAX
//     is chosen at init so that every chunk's nonzeros fit NZCAP);
//   * a row group (LPR lanes x VPL double2 = the K columns) issues all gathers of its row (up to
//     8 per batch) and its own x_i before the fma chain;
//   * xoff = gather offsets precomputed at init in double2 units -- local row * K/2 (>= 0), or
//     -1 - halo row * K/2 for halo rows (row partition) -- so a gather is one IMAD.WIDE + LDG.128;
//   * W is written with streaming stores (evict-first) so it does not push X out of L2.
// Each output w_ij is the fma chain over the row's nonzeros in ascending CSR order -- the oracle's
// chain, so W is bit-identical to the oracle given identical X (P3).  alpha / g: 8-row
// FP64 blocks merged into double-double accumulators in shared memory; fixed-order CTA reduction,
// one slot per CTA: ws.ag[(blockIdx.x * K + j) * 4 + {a_hi, a_lo, g_hi, g_lo}].
// UN = gathers per batch = the matrix's typical row length (chosen at init from {5, 7, 8}): a batch
// sized to the row keeps every register of x[UN] useful (cfg4 5-point rows: UN=5, 0.142 vs 0.188 ms
// at UN=8; cfg5 7-point rows: UN=7, 2.34 vs 2.75 ms), which is what lets 4 CTAs / SM fit at k <= 64.
template <int K, int UN_ = 8, int LPR_ = 0, int MINB_ = 0>
struct GatherCfg {
  static constexpr int LPR = LPR_ ? LPR_ : (K / 2 < 32 ? K / 2 : 32);   // lanes per row
  static constexpr int VPL = K / (2 * LPR);              // double2 per lane
  static constexpr int RG = 256 / LPR;                   // rows in flight per CTA
  static constexpr int RMAX = VPL > 1 ? (RG * 4 < 64 ? RG * 4 : 64) : (RG * 8 > 256 ? 256 : RG * 8);   // measured best at cfg4 / cfg5
  static constexpr int NZCAP = RMAX * 8 < 1024 ? RMAX * 8 : 1024;
  static constexpr int UN = UN_;                         // gathers per batch
  static constexpr int MINB = MINB_ ? MINB_ : (K >= 128 ? 2 : (UN <= 5 ? 4 : 3));
};

RF_DEV double2 ldg2_at(const char* base, uint32_t idx2) {   // base + idx2 double2s (one IMAD.WIDE.U32)
  return __ldg(reinterpret_cast<const double2*>(base + (uint64_t)idx2 * 16u));
}

// Chunk order (ord.x > 0, single rank): a matrix whose nonzeros sit at row offsets {1, d2, d3}
// (a 3-D stencil in lexicographic order: d2 = one grid line, d3 = one plane) is swept in tiles of
// ord.z lines across all planes -- position q -> (tile, plane, line in tile, chunk in line) --
// so a row's +-d3 neighbours are gathered a few chunks apart instead of 2 d3 rows apart (which
// exceeds L2 at cfg5: X was read 1.7x).  ord = (chunks per line, lines per plane, lines per tile,
// planes); chunk positions past the matrix are skipped.  W and every fma chain are unchanged.
RF_DEV int64_t chunk_of(int64_t q, int4 ord) {   // (positions < 2^31: 32-bit index arithmetic)
  if (ord.x == 0) return q;
  const uint32_t qq = (uint32_t)q;
  const uint32_t cx = qq % (uint32_t)ord.x;
  uint32_t r = qq / (uint32_t)ord.x;
  const uint32_t yy = r % (uint32_t)ord.z;
  r /= (uint32_t)ord.z;
  const uint32_t z = r % (uint32_t)ord.w, tb = r / (uint32_t)ord.w;
  const uint32_t y = tb * (uint32_t)ord.z + yy;
  return y < (uint32_t)ord.y ? ((int64_t)z * ord.y + y) * ord.x + cx : -1;
}
RF_DEV int64_t chunk_positions(int64_t nchunk, int4 ord) {
  return ord.x == 0 ? nchunk : (int64_t)((ord.y + ord.z - 1) / ord.z) * ord.z * ord.w * ord.x;
}

// requires n_loc * K / 2 < 2^31 and halo rows * K / 2 < 2^31 (checked at init).  (Measured and
// dropped: L1 prefetch of the next row's gathers, two rows per group in flight -- both slower.)
template <int K, bool HALO, int UN_ = 8, int LPR_ = 0, int MINB_ = 0>
__global__ void __launch_bounds__(256, GatherCfg<K, UN_, LPR_, MINB_>::MINB) spmm_gather_kernel(
    Ws ws, const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ xoff, const double* __restrict__ val,
    const double* __restrict__ Xloc, const int R, const double* __restrict__ Xown,   // gathered rows / own rows
    const int4 ord) {
  using C = GatherCfg<K, UN_, LPR_, MINB_>;
  constexpr int LPR = C::LPR, VPL = C::VPL, RG = C::RG, RMAX = C::RMAX, NZCAP = C::NZCAP, UN = C::UN, K2 = K / 2;
  __shared__ int32_t s_rp[3][RMAX + 1];
  __shared__ int32_t s_off[2][NZCAP];
  __shared__ double s_v[2][NZCAP];
  __shared__ dd s_acc[4 * VPL][256];
  griddep_wait();   // (programmatic dependent launch: the predecessor's writes are visible after this)
  if (*ws.status != ST_OK) return;
  const int tid = threadIdx.x, grp = tid / LPR, l = tid % LPR;
  const int64_t n = ws.n_loc, G = gridDim.x;
  const int64_t nchunk = (n + R - 1) / R;
  const int64_t npos = chunk_positions(nchunk, ord);
  const int T = (int)((npos - blockIdx.x + G - 1) / G);
  const char* Xb = reinterpret_cast<const char*>(Xloc);
  const char* Xo = reinterpret_cast<const char*>(Xown);
  const char* Hb = reinterpret_cast<const char*>(ws.halo);
  char* Wb = reinterpret_cast<char*>(ws.W);
  // chunk at position t G + blockIdx.x, or -1 (padding / past the matrix); computed once per
  // position (rolling ids of positions t, t + 1, t + 2 in registers)
  auto pos_id = [=](int t) -> int64_t {
    if (t >= T) return -1;
    const int64_t id = chunk_of((int64_t)t * G + blockIdx.x, ord);
    return id < nchunk ? id : (int64_t)-1;
  };
  auto r0_of = [=](int64_t id) { return id < 0 ? (int64_t)0 : id * R; };
  auto nr_of = [=](int64_t id) { return id < 0 ? 0 : (int)min((int64_t)R, n - id * R); };
  auto stage_rp = [&](int t, int64_t id) {
    if (t >= T) return;
    const int nr = nr_of(id);
    const int32_t* g = row_ptr + r0_of(id);
    int32_t* d = s_rp[t % 3];
    for (int i = tid; i <= nr; i += 256)
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(smem_u32(d + i)), "l"(g + i));
  };
  auto stage_nz = [&](int t, int64_t id) {   // needs s_rp[t % 3]
    if (t >= T) return;
    const int32_t* r = s_rp[t % 3];
    const int32_t p0 = r[0], cnt = r[nr_of(id)] - p0;
    for (int i = tid; i < cnt; i += 256) {
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(smem_u32(&s_off[t & 1][i])), "l"(xoff + p0 + i));
      cp_async8(&s_v[t & 1][i], val + p0 + i, true);
    }
  };
#pragma unroll
  for (int q = 0; q < 4 * VPL; ++q) s_acc[q][tid] = dd{0.0, 0.0};
  int64_t id_c = pos_id(0), id_n = pos_id(1);
  stage_rp(0, id_c);
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  stage_nz(0, id_c);
  stage_rp(1, id_n);
  cp_async_commit();
  double ba[2 * VPL], bg[2 * VPL];
#pragma unroll
  for (int u = 0; u < 2 * VPL; ++u) ba[u] = bg[u] = 0.0;
  int nb8 = 0;
  const double shift = ws.shift;
  for (int t = 0; t < T; ++t) {
    cp_async_wait<0>();
    __syncthreads();
    const int64_t id_nn = pos_id(t + 2);
    stage_nz(t + 1, id_n);   // row_ptr of chunk t+1 arrived with the previous group
    stage_rp(t + 2, id_nn);
    cp_async_commit();
    const int32_t* r = s_rp[t % 3];
    const int nr = nr_of(id_c);
    const int32_t p0 = r[0];
    const uint32_t rb2 = (uint32_t)r0_of(id_c) * K2 + l;   // double2 index of (chunk row 0, this lane)
    id_c = id_n;
    id_n = id_nn;
    const int32_t* so = s_off[t & 1];
    const double* sv = s_v[t & 1];
    auto gather = [&](int32_t off, int v) -> double2 {
      return (!HALO || off >= 0) ? ldg2_at(Xb + 16 * LPR * v, (uint32_t)off + l)
                                 : ldg2_at(Hb + 16 * LPR * v, (uint32_t)(-1 - off) + l);
    };
    // epilogue of one row: shift, streaming store of w_i, alpha / g block partials
    auto finish_row = [&](uint32_t i2, const double2 (&xi)[VPL], const double (&acc)[2 * VPL]) {
#pragma unroll
      for (int v = 0; v < VPL; ++v) {
        double w0 = acc[2 * v], w1 = acc[2 * v + 1];
        if (shift != 0.0) { w0 = __fma_rn(-shift, xi[v].x, w0); w1 = __fma_rn(-shift, xi[v].y, w1); }
        __stcs(reinterpret_cast<double2*>(Wb + 16 * LPR * v + (uint64_t)i2 * 16u), make_double2(w0, w1));
        ba[2 * v] = __fma_rn(xi[v].x, xi[v].x, ba[2 * v]);
        ba[2 * v + 1] = __fma_rn(xi[v].y, xi[v].y, ba[2 * v + 1]);
        bg[2 * v] = __fma_rn(xi[v].x, w0, bg[2 * v]);
        bg[2 * v + 1] = __fma_rn(xi[v].y, w1, bg[2 * v + 1]);
      }
      if (++nb8 == 8) {   // 8-row FP64 blocks merged into double-double
        nb8 = 0;
#pragma unroll
        for (int u = 0; u < 2 * VPL; ++u) {
          dd_add1(s_acc[u][tid], ba[u]); dd_add1(s_acc[2 * VPL + u][tid], bg[u]);
          ba[u] = bg[u] = 0.0;
        }
      }
    };
    for (int rl = grp; rl < nr; rl += RG) {
      {
        const int rr = rl;
        const int q0 = r[rr] - p0, q1 = r[rr + 1] - p0;
        const uint32_t i2 = rb2 + (uint32_t)rr * K2;
        double2 xi[VPL];
#pragma unroll
        for (int v = 0; v < VPL; ++v) xi[v] = ldg2_at(Xo + 16 * LPR * v, i2);
        double acc[2 * VPL];
#pragma unroll
        for (int u = 0; u < 2 * VPL; ++u) acc[u] = 0.0;
        for (int qb = q0; qb < q1; qb += UN) {   // all gathers of a batch issued before its fma chain
          const int cnt = q1 - qb;
          double2 x[UN][VPL];
#pragma unroll
          for (int u = 0; u < UN; ++u)
            if (u < cnt) {
              const int32_t off = so[qb + u];
#pragma unroll
              for (int v = 0; v < VPL; ++v) x[u][v] = gather(off, v);
            }
#pragma unroll
          for (int u = 0; u < UN; ++u)
            if (u < cnt) {
              const double vv = sv[qb + u];
#pragma unroll
              for (int v = 0; v < VPL; ++v) {
                acc[2 * v] = __fma_rn(vv, x[u][v].x, acc[2 * v]);
                acc[2 * v + 1] = __fma_rn(vv, x[u][v].y, acc[2 * v + 1]);
              }
            }
        }
        finish_row(i2, xi, acc);
      }
    }
  }
  cp_async_wait<0>();
#pragma unroll
  for (int u = 0; u < 2 * VPL; ++u) { dd_add1(s_acc[u][tid], ba[u]); dd_add1(s_acc[2 * VPL + u][tid], bg[u]); }
  __syncthreads();
  // fixed-order reduction over the RG row groups; thread grp * LPR + l owns columns 2 (l + LPR v) + {0, 1}
  for (int j = tid; j < K; j += 256) {
    const int pair = j >> 1, e = j & 1, v = pair / LPR, lj = pair % LPR;
    const int ua = 2 * v + e, ug = 2 * VPL + 2 * v + e;
    dd ta = s_acc[ua][lj], tg = s_acc[ug][lj];
    for (int g = 1; g < RG; ++g) { dd_add(ta, s_acc[ua][g * LPR + lj]); dd_add(tg, s_acc[ug][g * LPR + lj]); }
    double* slot = ws.ag + ((int64_t)blockIdx.x * K + j) * 4;
    slot[0] = ta.hi; slot[1] = ta.lo; slot[2] = tg.hi; slot[3] = tg.lo;
  }
}

// xoff for spmm_gather_kernel: gather offset of every local nonzero in double2 units
__global__ void spmm_xoff_kernel(const int32_t* __restrict__ col_idx, int64_t nnz, int64_t row0, int64_t row1,
                                 int64_t halo_lo, int k2, int32_t* __restrict__ xoff) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nnz; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t col = col_idx[q];
    int64_t o;
    if (col >= row0 && col < row1) o = (col - row0) * k2;
    else o = -1 - ((col < row0) ? col - halo_lo : (row0 - halo_lo) + (col - row1)) * k2;
    xoff[q] = (int32_t)o;
  }
}

}  // namespace rf
