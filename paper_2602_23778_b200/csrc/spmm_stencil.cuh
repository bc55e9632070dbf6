// spmm_stencil.cuh -- S1 (W = (A - shift I) X^, Alg. 4 line 1; Sec. 5.1 shift
// PAPER.md:1203) for CSR matrices whose nonzeros couple each point of a regular 2-D / 3-D grid only
// with itself and its axis neighbours (the configs' anisotropic Laplacians), with the
// X rows staged in shared memory by TMA instead of gathered from L2.
//
// Why: the gather kernel (spmm_csr.cuh) reads every nonzero's X row through L1/L2 -- nnz k 8 bytes
// (29 GB at cfg5, 1.3 GB at cfg4) against 8.7 / 0.6 GB of algorithmic HBM traffic -- and runs at
// the L2 throughput / gather-latency limit (58-63 % of HBM).  Here a CTA owns a pencil: a tile of
// L lines x R points of the (x, y) grid and KC of the k columns, swept along z (the slowest grid
// axis; a 2-D grid is swept along y with L = 1).  Each z-slab of the tile's footprint (the tile plus
// a one-point halo in x and y) is loaded ONCE by one 4-D TMA box (cp.async.bulk.tensor, zero fill
// outside the grid) into a 4-slot ring, two slabs ahead of the compute; a row's +-z neighbours are
// the same box position in the previous / next slot.  X therefore crosses L2 -> SM about
// (L + 2)(R + 2) / (L R) times instead of nnz / n times, and the kernel streams HBM.
//
// The nonzeros are re-packed once at init (refine_init_csr; A is borrowed and constant) into
// per-slab blocks of fixed-size row records -- NZR values in CSR order plus one 64-bit word of
// neighbour codes and the row length -- so a slab's records arrive with one bulk copy on the same
// mbarrier as its X box.  Each w_ij is the fma chain over the row's nonzeros in ascending CSR order
// (the oracle's chain, bit-identical W), shifted by fma(-shift, x_ij, .); alpha / g partials are
// 8-row FP64 blocks merged into double-double accumulators (same class as the gather kernel), one
// slot per CTA and column block, reduced in fixed order: deterministic.
#pragma once
#include <cuda.h>
#include <type_traits>   // CUtensorMap (encoded on the host through the driver entry point)

#include "common.cuh"

namespace rf {

constexpr int ST_THREADS = 512;     // 16 warps; thread 0 also issues the TMA loads
constexpr int ST_BLOCK = ST_THREADS;
constexpr int ST_SLOTS = 4;         // ring: slabs z - 1, z, z + 1 in use, z + 2 loading
constexpr int ST_WARPS = ST_THREADS / 32;

// codes of a nonzero's column relative to its row (x fastest, then y, then z)
enum : int { SC_SELF = 0, SC_XM, SC_XP, SC_YM, SC_YP, SC_ZM, SC_ZP };
constexpr uint64_t ST_CANON = 1ull << 55;   // code-word flag: canonical full stencil row (fast path)
constexpr uint64_t ST_SLAB_CANON = 1ull << 54;   // on record 0 of a slab block: every in-grid row canonical

struct StencilGeo {
  int nx, ny, nz;         // grid; a 2-D grid is (nx, 1, ny)
  int hy;                 // 1 if ny > 1: the box carries one halo line on each side
  int R, L, Rb, Lb;       // tile R points x L lines; box (R + 2) x (L + 2 hy)
  int ntx, nty, nseg, zlen;
  int nq, KC;             // column blocks of KC columns
  int nzr;                // values per row record (5 or 7)
  int mrg;                // slabs per FP64 alpha / g block (block = mrg x rows per thread per slab <= 8)
  int64_t d2, d3;         // row strides of y and z
  int box_bytes, meta_bytes, slot_bytes;
  int64_t blocks;         // metadata blocks (ntx nty nz)
};

// one record per output row: NZR values (CSR order) then a code word: byte u < NZR = code of
// nonzero u, byte 7 = row length (0 for padding rows of partial tiles)
template <int NZR>
__global__ void stencil_pack_kernel(const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                    const double* __restrict__ val, StencilGeo g, double* __restrict__ meta) {
  const int64_t n = (int64_t)g.nx * g.ny * g.nz;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int x = (int)(i % g.nx), y = (int)((i / g.nx) % g.ny), z = (int)(i / g.d3);
    const int tx = x / g.R, ty = y / g.L, lx = x % g.R, ly = y % g.L;
    const int64_t blk = ((int64_t)z * g.nty + ty) * g.ntx + tx;
    double* rec = meta + (blk * g.L * g.R + (int64_t)ly * g.R + lx) * (NZR + 1);
    uint64_t code = 0;
    const int32_t p0 = rp[i], p1 = rp[i + 1];
    for (int32_t p = p0; p < p1; ++p) {
      const int64_t o = (int64_t)ci[p] - i;
      const int c = o == 0 ? SC_SELF : o == -1 ? SC_XM : o == 1 ? SC_XP : o == -g.d2 ? SC_YM : o == g.d2 ? SC_YP
                  : o == -g.d3 ? SC_ZM : SC_ZP;
      rec[p - p0] = val[p];
      code |= (uint64_t)c << (8 * (p - p0));
    }
    code |= (uint64_t)(p1 - p0) << 56;
    // canonical full row: every neighbour present, in ascending column order -- 3-D (NZR = 7)
    // z-, y-, x-, self, x+, y+, z+; 2-D (NZR = 5) y-, x-, self, x+, y+ (y is the swept axis, codes ZM / ZP)
    const uint64_t canon = NZR == 7 ? 0x06040200010305ull : 0x0602000105ull;
    const uint64_t cmask = NZR == 7 ? 0xffffffffffffffull : 0xffffffffffull;
    if (p1 - p0 == NZR && (code & cmask) == canon) code |= ST_CANON;
    rec[NZR] = __longlong_as_double((long long)code);
  }
}

// per slab block: ST_SLAB_CANON on record 0 if every in-grid row of the block is canonical (padding
// rows of partial tiles have length 0 and are skipped by the kernel's bounds test)
template <int NZR>
__global__ void stencil_flag_kernel(StencilGeo g, double* __restrict__ meta) {
  for (int64_t blk = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; blk < g.blocks; blk += (int64_t)gridDim.x * blockDim.x) {
    double* rec = meta + blk * g.L * g.R * (NZR + 1);
    bool all = true;
    for (int r = 0; r < g.L * g.R; ++r) {
      const uint64_t code = (uint64_t)__double_as_longlong(rec[r * (NZR + 1) + NZR]);
      if ((code >> 56) != 0 && !(code & ST_CANON)) all = false;
    }
    if (all) rec[NZR] = __longlong_as_double((long long)((uint64_t)__double_as_longlong(rec[NZR]) | ST_SLAB_CANON));
  }
}

// structure check over all nonzeros: every offset is 0, +-1 (same line), +-d2 (same plane) or
// +-d3, and every row has at most 7 nonzeros.  bad[0] |= 1 on a violation; bad[1] = max row length.
__global__ void stencil_check_kernel(const int32_t* __restrict__ rp, const int32_t* __restrict__ ci, int64_t n,
                                     int64_t nx, int64_t d2, int64_t d3, int* bad) {
  int mx = 0, b = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t p0 = rp[i], p1 = rp[i + 1];
    mx = max(mx, p1 - p0);
    for (int32_t p = p0; p < p1; ++p) {
      const int64_t c = ci[p], o = c - i;
      bool ok;
      if (o == 0) ok = true;
      else if (o == 1 || o == -1) ok = (c / nx) == (i / nx);                   // no wrap across lines
      else if (d3 != d2 && (o == d2 || o == -d2)) ok = (c / d3) == (i / d3);   // 3-D: no wrap across planes
      else ok = (o == d3 || o == -d3);
      if (p > p0 && ci[p] <= ci[p - 1]) ok = false;                           // sorted, no duplicates
      if (!ok) b = 1;
    }
  }
  if (b) atomicOr(bad, 1);
  atomicMax(bad + 1, mx);
}

template <int KC, int NZR, bool SHIFT>
__global__ void __launch_bounds__(ST_BLOCK, 1) spmm_stencil_kernel(Ws ws, const __grid_constant__ CUtensorMap tmX,
                                                                   const double* __restrict__ meta, const StencilGeo g) {
  // a row's KC columns: LPR lanes x VPL double2, lane l owning double2 l + LPR v (each LDS.128 of a
  // quarter warp then reads 128 contiguous bytes of one row: no bank conflicts)
  constexpr int LPR = KC >= 16 ? 8 : KC / 2;
  constexpr int VPL = KC / (2 * LPR);
  constexpr int NV = 2 * VPL;                 // columns per thread
  constexpr int RGP = ST_THREADS / LPR;       // rows per pass
  constexpr int GPW = 32 / LPR;               // row groups per warp (lanes with equal l share columns)
  constexpr int REC = NZR + 1;
  // alpha / g: every g.mrg slabs the 2 NV per-thread FP64 block sums [ba | bg] are combined over the
  // warp's GPW row groups by a fixed xor butterfly on the lane bits 16, 8, .., LPR: the first SS stages
  // reduce-scatter (each keeps half), the remaining RB stages reduce into the lower group; each thread
  // then adds its NKEEP values into double-double accumulators (values NKEEP (gi >> RB) + j).
  constexpr int LOG_GPW = GPW == 1 ? 0 : GPW == 2 ? 1 : GPW == 4 ? 2 : GPW == 8 ? 3 : 4;
  constexpr int LOG_2NV = NV == 1 ? 1 : NV == 2 ? 2 : NV == 4 ? 3 : 4;
  constexpr int SS = LOG_GPW < LOG_2NV ? LOG_GPW : LOG_2NV;
  constexpr int RB = LOG_GPW - SS;
  constexpr int NKEEP = (2 * NV) >> SS;
  extern __shared__ __align__(128) unsigned char st_smem[];
  uint64_t* mbar = reinterpret_cast<uint64_t*>(st_smem);           // full[slot]: box + records landed
  int* done = reinterpret_cast<int*>(st_smem + 64);                 // warps through iteration m (slot m % 4)
  unsigned char* slots = st_smem + 128;
  griddep_wait();   // (programmatic dependent launch: the predecessor's writes are visible after this)
  if (*ws.status != ST_OK) return;
  const int tid = threadIdx.x, grp = tid / LPR, l = tid % LPR, lane = tid & 31;
  const int K = ws.k, nq = g.nq;
  const int q = blockIdx.x % nq, b = blockIdx.x / nq, nb = gridDim.x / nq;
  // Work split (per column block, nb CTAs): R = pencils / nb full rounds -- round j gives CTA b the whole
  // z extent of pencil b + nb j, so neighbouring CTAs sweep neighbouring pencils in step and share their x /
  // y halo boxes in L2 -- then the pencils mod nb remaining pencils as nb equal contiguous ranges of slabs
  // (pencil-major), so every CTA computes the same number of slabs (+-1).  (Fixed z segments dealt
  // round-robin left 4 CTAs with a 12th segment while 32 had 11 at cfg5: 7 % of the kernel idle.)
  const int64_t PEN = (int64_t)g.ntx * g.nty;
  const int64_t NR = PEN / nb;
  const int64_t Sr = (PEN - NR * nb) * g.nz, rs0 = Sr * b / nb, rs1 = Sr * (b + 1) / nb;
  if (tid == 0) {
    for (int s = 0; s < ST_SLOTS; ++s) { mbar_init(&mbar[s], 1); done[s] = 0; }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  // the CTA's load sequence: items it = 0, 1, .. -> (pencil, z range [zs, ze)); loads z = zs - 1 .. ze
  struct Cur { int64_t it; int z, zs, ze, tx, ty; };
  auto item_exists = [&](int64_t it) -> bool {
    return it < NR || (rs0 < rs1 && (rs0 / g.nz + (it - NR)) * g.nz < rs1);
  };
  auto item_begin = [&](Cur& c) -> bool {
    if (!item_exists(c.it)) return false;
    int64_t p;
    if (c.it < NR) {
      p = b + nb * c.it;
      c.zs = 0;
      c.ze = g.nz;
    } else {
      const int64_t t = rs0 / g.nz + (c.it - NR), base = t * g.nz;
      p = NR * nb + t;
      c.zs = (int)(rs0 > base ? rs0 - base : 0);
      c.ze = (int)(rs1 - base < g.nz ? rs1 - base : g.nz);
    }
    c.tx = (int)(p % g.ntx);
    c.ty = (int)(p / g.ntx);
    c.z = c.zs - 1;
    return true;
  };
  auto advance = [&](Cur& c) -> bool {   // next load; false when the sequence ends
    if (++c.z <= c.ze) return true;
    ++c.it;
    return item_begin(c);
  };
  auto issue = [&](const Cur& c, int m) {   // one lane 0: load m of the sequence into slot m % 4
    const int s = m % ST_SLOTS;
    // (the slot was last read by generic-proxy loads, ordered before this thread by the counter:
    //  order them before the async-proxy TMA / bulk writes that refill it)
    fence_async_smem();
    unsigned char* sl = slots + (size_t)s * g.slot_bytes;
    const bool inner = c.z >= c.zs && c.z < c.ze;
    mbar_expect_tx(&mbar[s], g.box_bytes + (inner ? g.meta_bytes : 0));
    tma_load_4d(sl, &tmX, q * KC, c.tx * g.R - 1, c.ty * g.L - g.hy, c.z, &mbar[s]);
    if (inner) {
      const int64_t blk = ((int64_t)c.z * g.nty + c.ty) * g.ntx + c.tx;
      bulk_g2s(sl + g.box_bytes, meta + blk * g.L * g.R * REC, g.meta_bytes, &mbar[s]);
    }
  };

  // No CTA-wide barrier per slab: the slot of load m - 1 (read as X+ / X0 / X- by iterations m - 2 .. m)
  // is refilled with load m + 3 by the LAST warp to finish iteration m (a shared counter per slot);
  // every lane 0 tracks the load sequence so whichever warp is last can issue.
  Cur cons{0, 0, 0, 0, 0, 0}, prod{0, 0, 0, 0, 0, 0};
  bool more_c = item_begin(cons);
  bool more_p = item_begin(prod);
  int m_issued = 0;
  if (lane == 0) {
    for (int t = 0; t < 3 && more_p; ++t) {
      if (tid == 0) issue(prod, m_issued);
      ++m_issued;
      more_p = advance(prod);
    }
  }
  const double shift = ws.shift;
  const int RbKC = g.Rb * KC;
  const int nrow = g.L * g.R;
  // per-thread constants of the tile walk: the first row (ly0, lx0) and the per-pass step (dly, dlx)
  const int ly0 = grp / g.R, lx0 = grp - ly0 * g.R;
  const int dly = RGP / g.R, dlx = RGP - dly * g.R;
  const int64_t d2K = g.d2 * K, d3K = g.d3 * K;
  const int d2i = (int)g.d2;
  double ba[NV], bg[NV];
  dd acc_dd[NKEEP];
#pragma unroll
  for (int u = 0; u < NV; ++u) ba[u] = bg[u] = 0.0;
#pragma unroll
  for (int u = 0; u < NKEEP; ++u) acc_dd[u] = dd{0.0, 0.0};
  auto merge = [&]() {
    double v[2 * NV];
#pragma unroll
    for (int u = 0; u < NV; ++u) { v[u] = ba[u]; v[NV + u] = bg[u]; ba[u] = bg[u] = 0.0; }
#pragma unroll
    for (int st = 0; st < LOG_GPW; ++st) {
      const int m = 16 >> st;
      const bool hi = (lane & m) != 0;
      if (st < SS) {                       // reduce-scatter: keep half n of the values
        const int n = (2 * NV) >> (st + 1);
#pragma unroll
        for (int j = 0; j < NV; ++j) {
          if (j < n) {
            const double keep = hi ? v[n + j] : v[j], send = hi ? v[j] : v[n + j];
            const double other = __shfl_xor_sync(0xffffffffu, send, m);
            v[j] = hi ? __dadd_rn(other, keep) : __dadd_rn(keep, other);   // the lower group's value first
          }
        }
      } else {                             // reduce into the lower group
#pragma unroll
        for (int j = 0; j < NKEEP; ++j) {
          const double other = __shfl_xor_sync(0xffffffffu, v[j], m);
          v[j] = hi ? 0.0 : __dadd_rn(v[j], other);
        }
      }
    }
#pragma unroll
    for (int j = 0; j < NKEEP; ++j) dd_add1(acc_dd[j], v[j]);
  };
  int mrg = 0;
  double* const W = ws.W;
  if (more_c) mbar_wait(&mbar[0], 0);
  for (int m = 0; more_c; ++m) {
    const int nxt = m + 1;                     // every thread waits each load once, in order
    const bool has_next = !(cons.z == cons.ze && !item_exists(cons.it + 1));
    if (has_next) mbar_wait(&mbar[nxt % ST_SLOTS], (nxt / ST_SLOTS) & 1);
    if (cons.z >= cons.zs && cons.z < cons.ze) {   // compute the outputs of slab z
      const double* X0 = reinterpret_cast<const double*>(slots + (size_t)(m % ST_SLOTS) * g.slot_bytes);
      const double* Xm = reinterpret_cast<const double*>(slots + (size_t)((m + 3) % ST_SLOTS) * g.slot_bytes);
      const double* Xp = reinterpret_cast<const double*>(slots + (size_t)((m + 1) % ST_SLOTS) * g.slot_bytes);
      const double* rec0 = reinterpret_cast<const double*>(reinterpret_cast<const unsigned char*>(X0) + g.box_bytes);
      const int x0 = cons.tx * g.R, y0 = cons.ty * g.L;
      const int xlim = g.nx - x0, ylim = g.ny - y0;   // rows of the tile inside the grid: lx < xlim, ly < ylim
      // W at (x0, y0, z), this thread's columns
      double* const wz = W + ((int64_t)cons.z * d3K + (int64_t)y0 * d2K + (int64_t)x0 * K + q * KC + 2 * l);
      // rows of the slab; ALL: every in-grid row of this slab block is a canonical full stencil row
      // (flag on record 0, set at init), so no row waits on its code word before its neighbour loads
      auto rows = [&](auto all_canon) {
      int ly = ly0, lx = lx0;
      for (int rr = grp; rr < nrow; rr += RGP) {
        const int cly = ly, clx = lx;
        lx += dlx; ly += dly;
        if (lx >= g.R) { lx -= g.R; ++ly; }
        if (clx >= xlim || cly >= ylim) continue;
        const double2* rv = reinterpret_cast<const double2*>(rec0 + rr * REC);
        double vv[REC];
#pragma unroll
        for (int u = 0; u < REC / 2; ++u) { const double2 t = rv[u]; vv[2 * u] = t.x; vv[2 * u + 1] = t.y; }
        const int ctr = ((cly + g.hy) * g.Rb + clx + 1) * KC + 2 * l;
        double acc[NV];
#pragma unroll
        for (int u = 0; u < NV; ++u) acc[u] = 0.0;
        auto nz = [&](double val, const double* p) {   // acc += val * (this lane's part of row p)
#pragma unroll
          for (int v = 0; v < VPL; ++v) {
            const double2 t = *reinterpret_cast<const double2*>(p + 2 * LPR * v);
            acc[2 * v] = __fma_rn(val, t.x, acc[2 * v]);
            acc[2 * v + 1] = __fma_rn(val, t.y, acc[2 * v + 1]);
          }
        };
        const double* xc = X0 + ctr;
        double2 xi[VPL];         // this row's own x (the diagonal nonzero's operand, and alpha / g)
#pragma unroll
        for (int v = 0; v < VPL; ++v) xi[v] = *reinterpret_cast<const double2*>(xc + 2 * LPR * v);
        auto nzc = [&](double val) {   // acc += val * x_i (registers)
#pragma unroll
          for (int v = 0; v < VPL; ++v) {
            acc[2 * v] = __fma_rn(val, xi[v].x, acc[2 * v]);
            acc[2 * v + 1] = __fma_rn(val, xi[v].y, acc[2 * v + 1]);
          }
        };
        const uint64_t code = decltype(all_canon)::value ? ST_CANON : (uint64_t)__double_as_longlong(vv[NZR]);
        if (code & ST_CANON) {   // the fma chain in CSR (= ascending column) order, offsets fixed
          if constexpr (NZR == 7) {
            nz(vv[0], Xm + ctr); nz(vv[1], xc - RbKC); nz(vv[2], xc - KC); nzc(vv[3]);
            nz(vv[4], xc + KC); nz(vv[5], xc + RbKC); nz(vv[6], Xp + ctr);
          } else {
            nz(vv[0], Xm + ctr); nz(vv[1], xc - KC); nzc(vv[2]); nz(vv[3], xc + KC); nz(vv[4], Xp + ctr);
          }
        } else {                 // boundary rows: the coded neighbours, CSR order
          const int len = (int)(code >> 56);
          for (int u = 0; u < len; ++u) {
            const int c = (int)((code >> (8 * u)) & 0xff);
            const int o = c == SC_XM ? -KC : c == SC_XP ? KC : c == SC_YM ? -RbKC : c == SC_YP ? RbKC : 0;
            const double* base = c == SC_ZM ? Xm : c == SC_ZP ? Xp : X0;
            nz(rec0[rr * REC + u], base + ctr + o);
          }
        }
        double* wrow = wz + (cly * d2i + clx) * K;   // (d3 K < 2^31: checked at setup)
#pragma unroll
        for (int v = 0; v < VPL; ++v) {
          double w0 = acc[2 * v], w1 = acc[2 * v + 1];
          if constexpr (SHIFT) { w0 = __fma_rn(-shift, xi[v].x, w0); w1 = __fma_rn(-shift, xi[v].y, w1); }
          __stcs(reinterpret_cast<double2*>(wrow + 2 * LPR * v), make_double2(w0, w1));
          ba[2 * v] = __fma_rn(xi[v].x, xi[v].x, ba[2 * v]);
          ba[2 * v + 1] = __fma_rn(xi[v].y, xi[v].y, ba[2 * v + 1]);
          bg[2 * v] = __fma_rn(xi[v].x, w0, bg[2 * v]);
          bg[2 * v + 1] = __fma_rn(xi[v].y, w1, bg[2 * v + 1]);
        }
      }
      };
      if ((uint64_t)__double_as_longlong(rec0[NZR]) & ST_SLAB_CANON) rows(std::true_type{});
      else rows(std::false_type{});
      if (++mrg == g.mrg) { mrg = 0; merge(); }   // (warp-uniform: every thread walks the same slabs)
    }
    __syncwarp();                              // this warp's reads of iteration m are done
    if (lane == 0) {
      // (monotonic: ST_WARPS arrivals per use) last warp through iteration m: slot of load m - 1 is free
      if (stage_release_last(&done[m % ST_SLOTS], ST_WARPS) && more_p) issue(prod, m_issued);
      if (more_p) { ++m_issued; more_p = advance(prod); }
    }
    more_c = advance(cons);
  }
  merge();
  // fixed-order reduction over the warps, then this CTA's slot.  Thread (warp w, group gi, l) holds
  // values NKEEP (gi >> RB) + j (j < NKEEP) of [ba | bg] for its columns: value t < NV is alpha of column
  // u = t, else g of column u = t - NV; column u of lane l is 2 (l + LPR (u / 2)) + (u & 1).
  __syncthreads();
  dd* red = reinterpret_cast<dd*>(slots);              // [ST_WARPS][2 NV][LPR]
  {
    const int gi = lane / LPR;
    if ((gi & ((1 << RB) - 1)) == 0) {
#pragma unroll
      for (int j = 0; j < NKEEP; ++j) red[((tid >> 5) * 2 * NV + NKEEP * (gi >> RB) + j) * LPR + l] = acc_dd[j];
    }
  }
  __syncthreads();
  for (int t = tid; t < 2 * NV * LPR; t += ST_THREADS) {
    const int val = t / LPR, lj = t % LPR;
    dd tot = red[val * LPR + lj];
    for (int w = 1; w < ST_WARPS; ++w) dd_add(tot, red[(w * 2 * NV + val) * LPR + lj]);
    const int u = val < NV ? val : val - NV;
    const int j = 2 * (lj + LPR * (u / 2)) + (u & 1);   // column within the block
    double* slot = ws.ag + ((int64_t)b * K + q * KC + j) * 4 + (val < NV ? 0 : 2);
    slot[0] = tot.hi; slot[1] = tot.lo;
  }
}

}  // namespace rf
