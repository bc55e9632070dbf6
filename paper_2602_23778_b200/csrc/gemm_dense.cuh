// gemm_dense.cuh -- S1 for dense A: W = A X^ - shift X^ (Alg. 4 line 1, PAPER.md:434;
// Sec. 5.1 shift) on the FP64 tensor cores (DMMA.8x8x4), plus the
// S2 epilogue partials alpha_j = x_j^T x_j and g_j = x_j^T w_j (lines 3-4).
//
// Shape: M = n_loc rows of A (row-major, lda), N = k (padded to NT), K = n.
// A is streamed from HBM exactly once; X^ (n x k, 16 MiB at cfg3) stays L2-resident.
// CTA tile BM x NT, K step BK, STAGES-deep cp.async pipeline; warps tile the CTA
// output in WM x WN blocks of m8n8 DMMA fragments.  Split-K over gridDim.x (row tiles over
// gridDim.y, so a tile's splits are launched side by side and its fix-up overlaps later tiles) makes
// 148 SMs busy at cfg3 (256 row tiles x 4 splits = 1024 CTAs, 2 resident per SM); the
// split partials are summed in fixed order by the last CTA of each row tile (fused_finish), or by
// w_finish (deterministic either way).
#pragma once
#include <cuda.h>   // CUtensorMap

#include "common.cuh"

namespace rf {

template <int NT, int BM, int WM, int WN, int BK, int STAGES>
struct GemmCfg {
  static constexpr int WARPS_M = BM / WM, WARPS_N = NT / WN, WARPS = WARPS_M * WARPS_N;
  static constexpr int THREADS = WARPS * 32;
  static constexpr int LDA_S = BK + 4;                         // 8 rows x 4 cols frag reads: 2-way min
  static constexpr int LDB_S = NT + ((NT % 16 == 8) ? 0 : 8);  // 4 rows x 8 cols frag reads: 2-way min
  static constexpr int A_STAGE = BM * LDA_S, B_STAGE = BK * LDB_S;
  static constexpr int SMEM = STAGES * (A_STAGE + B_STAGE) * 8;
  static constexpr int MI = WM / 8, NI = WN / 8;
};

// Sum the S split partials of rows [rb, re) in fixed order s = 0..S-1, apply the shift
// (w = fma(-shift, x, w)), write W, and write the double-double partials of
// alpha_j = sum x_ij^2 and g_j = sum x_ij w_ij into alpha/g slot `slot` of Ws::ag.
// NTH threads (tid < NTH) take NTH / k rows side by side; sa, sg: NTH doubles-doubles of scratch.
// A fixed row range per slot and fixed orders everywhere: deterministic.
template <int NTH>
RF_DEV void tile_finish(const Ws& ws, const double* __restrict__ X, int nsplit, int64_t split_stride, int64_t rb,
                        int64_t re, int slot, int tid, dd* sa, dd* sg) {
  const int k = ws.k;
  const int R = NTH / k;                     // rows processed in parallel (k <= NTH)
  const int r = tid / k, j = tid % k;
  dd a = {0.0, 0.0}, g = {0.0, 0.0};
  if (r < R) {
    // 4 rows per step with every load issued before the sums (the row order of the dd accumulation
    // and the split order of each sum are unchanged: bit-identical to one row at a time)
    for (int64_t i0 = rb + r; i0 < re; i0 += 4 * R) {
      double w[4], x[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t i = i0 + u * R;
        const int64_t e = i * k + j;
        const bool ok = i < re;
        w[u] = ok ? (nsplit == 1 ? ws.W[e] : ws.Wpart[e]) : 0.0;
        x[u] = ok ? X[e] : 0.0;
      }
      // splits 1.. in batches of 4: every load of a batch in flight before its (split-ordered) sums
      // (4 x 4 values: the fused fix-up must stay within the GEMM main loop's register budget)
      for (int s0 = 1; s0 < nsplit; s0 += 4) {
        double p[4][4];
#pragma unroll
        for (int b = 0; b < 4; ++b)
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int64_t i = i0 + u * R;
            p[b][u] = (s0 + b < nsplit && i < re) ? ws.Wpart[(s0 + b) * split_stride + i * k + j] : 0.0;
          }
#pragma unroll
        for (int b = 0; b < 4; ++b)
          if (s0 + b < nsplit) {
#pragma unroll
            for (int u = 0; u < 4; ++u) w[u] = __dadd_rn(w[u], p[b][u]);
          }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t i = i0 + u * R;
        if (i < re) {
          double wv = w[u];
          if (ws.shift != 0.0) wv = __fma_rn(-ws.shift, x[u], wv);
          ws.W[i * k + j] = wv;
          dd_add_prod(a, x[u], x[u]);
          dd_add_prod(g, x[u], wv);
        }
      }
    }
  }
  sa[tid] = a;
  sg[tid] = g;
}
// second half of tile_finish, after a barrier over the NTH threads: the fixed-order sum over the R row groups
template <int NTH>
RF_DEV void tile_finish_slot(const Ws& ws, int slot, int tid, const dd* sa, const dd* sg) {
  const int k = ws.k, R = NTH / k;
  if (tid < k) {
    dd ta = sa[tid], tg = sg[tid];
    for (int q = 1; q < R; ++q) { dd_add(ta, sa[q * k + tid]); dd_add(tg, sg[q * k + tid]); }
    double* sl = ws.ag + ((int64_t)slot * k + tid) * 4;
    sl[0] = ta.hi; sl[1] = ta.lo; sl[2] = tg.hi; sl[3] = tg.lo;
  }
}
// Split-K fix-up fused into the GEMM (FusedFinish::on): every CTA stores its partial tile, the LAST of
// the nsplit CTAs of a row tile (a per-tile arrival counter; threadfence reduction) sums the partials
// in split order and does w_finish's work for the tile's rows into alpha/g slot = the row tile, then
// re-arms the counter.  Saves the w_finish launch and its second pass over the partials.
struct FusedFinish {
  Ws ws;                    // W, Wpart, shift, ag, k, n_loc
  const double* X;          // the shift operand (the sweep's X^)
  int* cnt;                 // per row-tile arrival counters (zero between launches)
  int on;
  // refine_sweep_host's overlapped upload (TMA GEMM only): X^ arrives in chunks of ready_rows rows on a
  // copy stream, each followed by a 4-byte copy of `epoch` into ready[chunk]; the producer waits for
  // the chunk of each K step before loading its X^ box, the fix-up for its tile's rows.  null: X^ resident
  const unsigned* ready;
  unsigned epoch;
  int ready_rows;
};
// wait until rows [r0, r1) of X^ have arrived (see FusedFinish::ready); then order the copy engine's
// writes before this thread's async-proxy (TMA) and generic reads
// (a failed upload never sets its flags: after 5 s the wait gives up and marks the sweep failed, rather
// than hanging the device)
RF_DEV void wait_rows(const FusedFinish& f, int64_t r0, int64_t r1) {
  if (f.ready == nullptr || r1 <= r0) return;
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;\n" : "=l"(t0));
  for (int64_t c = r0 / f.ready_rows; c <= (r1 - 1) / f.ready_rows; ++c) {
    unsigned v;
    while (true) {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(f.ready + c) : "memory");
      if (v == f.epoch) break;
      uint64_t t;
      asm volatile("mov.u64 %0, %%globaltimer;\n" : "=l"(t));
      if (t - t0 > 5000000000ull) {
        atomicCAS(f.ws.status, ST_OK, ST_DIVERGED);
        return;
      }
      __nanosleep(256);
    }
  }
  asm volatile("fence.proxy.async.global;\n" ::: "memory");
}
// called by the NTH consumer threads after their partial-tile stores; bar(): a barrier over them
template <int NTH, int BM, typename Bar>
RF_DEV void fused_finish(const FusedFinish& f, int nsplit, int64_t split_stride, int64_t m0, int tid, void* scratch,
                         int* s_flag, Bar bar) {
  __threadfence();                                  // this CTA's partial stores -> visible device-wide
  bar();
  if (tid == 0) {
    const int old = atomicAdd(&f.cnt[blockIdx.y], 1);
    *s_flag = (old == nsplit - 1);
    if (old == nsplit - 1) f.cnt[blockIdx.y] = 0;   // re-arm (every other split has arrived)
  }
  bar();
  if (!*s_flag) return;
  __threadfence();                                  // (acquire side of the counter)
  if (f.ready) {                                    // (overlapped upload: the tile's X^ rows)
    if (tid == 0) wait_rows(f, m0, (m0 + BM < f.ws.n_loc) ? m0 + BM : f.ws.n_loc);
    bar();
  }
  dd* sa = reinterpret_cast<dd*>(scratch);
  dd* sg = sa + NTH;
  const int64_t re = (m0 + BM < f.ws.n_loc) ? m0 + BM : f.ws.n_loc;
  tile_finish<NTH>(f.ws, f.X, nsplit, split_stride, m0, re, blockIdx.y, tid, sa, sg);
  bar();
  tile_finish_slot<NTH>(f.ws, blockIdx.y, tid, sa, sg);
}

// out[m][j] = sum_{l in [kb, ke)} A[m][l] X[l][j], m in [0, M), j in [0, k)
template <int NT, int BM, int WM, int WN, int BK, int STAGES>
__global__ void __launch_bounds__(GemmCfg<NT, BM, WM, WN, BK, STAGES>::THREADS)
gemm_ax_kernel(const double* __restrict__ A, int64_t lda, const double* __restrict__ X, int32_t k,
               int64_t M, int64_t K, int64_t kchunk, double* __restrict__ out, int64_t out_split_stride,
               int a_vec16, int b_vec16, const int* __restrict__ status, const FusedFinish fin) {
  using C = GemmCfg<NT, BM, WM, WN, BK, STAGES>;
  griddep_wait();   // (programmatic dependent launch: the predecessor's writes are visible after this)
  if (*status != ST_OK) return;
  extern __shared__ __align__(16) double smem[];
  double* As = smem;
  double* Bs = smem + STAGES * C::A_STAGE;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / C::WARPS_N, wn = warp % C::WARPS_N;
  const int64_t m0 = (int64_t)blockIdx.y * BM;   // row tile
  const int64_t kb = (int64_t)blockIdx.x * kchunk;   // split
  const int64_t ke = (kb + kchunk < K) ? kb + kchunk : K;
  const int nk = (int)((ke - kb + BK - 1) / BK);
  out += (int64_t)blockIdx.x * out_split_stride;

  // per-thread copy coordinates are the same for every stage: precompute them once
  constexpr int ACH16 = BM * BK / 2, BCH16 = BK * NT / 2;
  constexpr int AIT16 = (ACH16 + C::THREADS - 1) / C::THREADS, BIT16 = (BCH16 + C::THREADS - 1) / C::THREADS;
  auto load_stage = [&](int stage, int it) {
    const int64_t k0 = kb + (int64_t)it * BK;
    double* as = As + stage * C::A_STAGE;
    double* bs = Bs + stage * C::B_STAGE;
    if (a_vec16) {
#pragma unroll
      for (int q = 0; q < AIT16; ++q) {
        const int c = tid + q * C::THREADS;
        if (ACH16 % C::THREADS == 0 || c < ACH16) {
          const int r = c / (BK / 2), cc = (c % (BK / 2)) * 2;
          const int64_t gr = m0 + r, gc = k0 + cc;
          const bool ok = (gr < M) && (gc < ke);  // K and ke are even on this path
          cp_async16(as + r * C::LDA_S + cc, ok ? (const void*)(A + gr * lda + gc) : (const void*)A, ok);
        }
      }
    } else {
      for (int c = tid; c < BM * BK; c += C::THREADS) {
        const int r = c / BK, cc = c % BK;
        const int64_t gr = m0 + r, gc = k0 + cc;
        const bool ok = (gr < M) && (gc < ke);
        cp_async8(as + r * C::LDA_S + cc, ok ? (const void*)(A + gr * lda + gc) : (const void*)A, ok);
      }
    }
    if (b_vec16) {
#pragma unroll
      for (int q = 0; q < BIT16; ++q) {
        const int c = tid + q * C::THREADS;
        if (BCH16 % C::THREADS == 0 || c < BCH16) {
          const int r = c / (NT / 2), cc = (c % (NT / 2)) * 2;
          const int64_t gr = k0 + r;
          const bool ok = (gr < ke) && (cc < k);   // k even on this path
          cp_async16(bs + r * C::LDB_S + cc, ok ? (const void*)(X + gr * k + cc) : (const void*)X, ok);
        }
      }
    } else {
      for (int c = tid; c < BK * NT; c += C::THREADS) {
        const int r = c / NT, cc = c % NT;
        const int64_t gr = k0 + r;
        const bool ok = (gr < ke) && (cc < k);
        cp_async8(bs + r * C::LDB_S + cc, ok ? (const void*)(X + gr * k + cc) : (const void*)X, ok);
      }
    }
  };

  double acc[C::MI][C::NI][2];
#pragma unroll
  for (int i = 0; i < C::MI; ++i)
#pragma unroll
    for (int j = 0; j < C::NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nk) load_stage(s, s);
    cp_async_commit();
  }
  const int ar = wm * WM + (lane >> 2), ac = lane & 3;   // A frag coords within the tile
  const int br = lane & 3, bc = wn * WN + (lane >> 2);   // B frag coords
  for (int it = 0; it < nk; ++it) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {  // prefetch stage it + STAGES - 1 (its buffer was consumed at iteration it - 1)
      const int nx = it + STAGES - 1;
      if (nx < nk) load_stage(nx % STAGES, nx);
      cp_async_commit();
    }
    const double* as = As + (it % STAGES) * C::A_STAGE;
    const double* bs = Bs + (it % STAGES) * C::B_STAGE;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double a[C::MI], b[C::NI];
#pragma unroll
      for (int i = 0; i < C::MI; ++i) a[i] = as[(ar + i * 8) * C::LDA_S + kk + ac];
#pragma unroll
      for (int j = 0; j < C::NI; ++j) b[j] = bs[(kk + br) * C::LDB_S + bc + j * 8];
#pragma unroll
      for (int i = 0; i < C::MI; ++i)
#pragma unroll
        for (int j = 0; j < C::NI; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
  }
  cp_async_wait<0>();

  // epilogue: fragment (i, j) -> rows m0 + wm*WM + i*8 + lane/4, cols wn*WN + j*8 + 2*(lane%4) + {0,1}
#pragma unroll
  for (int i = 0; i < C::MI; ++i) {
    const int64_t r = m0 + wm * WM + i * 8 + (lane >> 2);
    if (r >= M) continue;
#pragma unroll
    for (int j = 0; j < C::NI; ++j) {
      const int c = wn * WN + j * 8 + 2 * (lane & 3);
      double* o = out + r * k + c;
      if (b_vec16 && c < k) {   // k even: c, c+1 both valid
        *reinterpret_cast<double2*>(o) = make_double2(acc[i][j][0], acc[i][j][1]);
      } else {
        if (c < k) o[0] = acc[i][j][0];
        if (c + 1 < k) o[1] = acc[i][j][1];
      }
    }
  }
  if (fin.on) {   // (the pipeline is drained: the stage buffers are free scratch)
    __shared__ int s_last;
    fused_finish<C::THREADS, BM>(fin, (int)gridDim.x, out_split_stride, m0, tid, smem, &s_last,
                                 [] { __syncthreads(); });
  }
}

// ---------------------------------------------------------------- TMA-fed variant (north_star "DMMA
// tiled kernel fed by TMA"): the same tiles, DMMA fragments and epilogue, but every stage of A and X^
// arrives by cp.async.bulk.tensor (SASS UTMALDG) issued by ONE producer warp into an STAGES-deep ring of
// 128-byte-swizzled boxes (16 doubles wide, so the 8-row x 4-column A fragment reads and 4-row x 8-column
// B fragment reads are bank-conflict free without padding), with full / empty mbarriers between the
// producer and the consumer warps -- no per-thread copy instructions or address arithmetic in the
// main loop.  Out-of-range rows / columns (ragged n_loc, K tail, k < NT) are zero-filled by the TMA
// unit.  Requires lda and k even (16-byte row strides) and 16-byte aligned A and X.
template <int NT, int BM, int BK>
struct GemmTmaCfg {
  static constexpr int A_BOXES = BK / 16, B_BOXES = NT / 16;
  static constexpr int A_BOX_BYTES = BM * 128, B_BOX_BYTES = BK * 128;
  static constexpr int STAGE_BYTES = A_BOXES * A_BOX_BYTES + B_BOXES * B_BOX_BYTES;
};
template <int NT, int BM, int WM, int WN, int BK, int STAGES>
__global__ void __launch_bounds__(GemmCfg<NT, BM, WM, WN, BK, STAGES>::THREADS + 32)
gemm_ax_tma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmX, int32_t k,
                   int64_t M, int64_t K, int64_t kchunk, double* __restrict__ out, int64_t out_split_stride,
                   const int* __restrict__ status, const FusedFinish fin) {
  using C = GemmCfg<NT, BM, WM, WN, BK, STAGES>;
  using T = GemmTmaCfg<NT, BM, BK>;
  static_assert(BK % 16 == 0 && NT % 16 == 0, "16-double TMA boxes");
  griddep_wait();   // (programmatic dependent launch: the predecessor's writes are visible after this)
  if (*status != ST_OK) return;
  extern __shared__ __align__(1024) unsigned char gsm[];
  // [STAGES x stage] ring (1024-byte aligned for the 128-byte swizzle), then the mbarriers
  unsigned char* ring = smem_align1024(gsm);
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + STAGES * T::STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t m0 = (int64_t)blockIdx.y * BM;   // row tile
  const int64_t kb = (int64_t)blockIdx.x * kchunk;   // split
  const int64_t ke = (kb + kchunk < K) ? kb + kchunk : K;
  const int nk = (int)((ke - kb + BK - 1) / BK);
  out += (int64_t)blockIdx.x * out_split_stride;
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], C::WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (warp == C::WARPS) {   // producer warp
    if (lane == 0) {
      for (int it = 0; it < nk; ++it) {
        const int s = it % STAGES;
        if (it >= STAGES) {
          mbar_wait(&empty[s], ((it / STAGES) - 1) & 1);
          // the consumers read stage s with generic-proxy loads; order them before the async-proxy
          // (TMA) writes that refill it
          fence_async_smem();
        }
        unsigned char* st = ring + s * T::STAGE_BYTES;
        const int k0 = (int)(kb + (int64_t)it * BK);
        mbar_expect_tx(&full[s], T::STAGE_BYTES);
#pragma unroll
        for (int b = 0; b < T::A_BOXES; ++b) tma_load_2d(st + b * T::A_BOX_BYTES, &tmA, k0 + 16 * b, (int)m0, &full[s]);
        wait_rows(fin, k0, (k0 + BK < K) ? k0 + BK : K);   // (overlapped upload only)
#pragma unroll
        for (int b = 0; b < T::B_BOXES; ++b)
          tma_load_2d(st + T::A_BOXES * T::A_BOX_BYTES + b * T::B_BOX_BYTES, &tmX, 16 * b, k0, &full[s]);
      }
    }
    return;
  }
  const int wm = warp / C::WARPS_N, wn = warp % C::WARPS_N;
  double acc[C::MI][C::NI][2];
#pragma unroll
  for (int i = 0; i < C::MI; ++i)
#pragma unroll
    for (int j = 0; j < C::NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const int ar = wm * WM + (lane >> 2), ac = lane & 3;   // A frag: rows ar + 8 i, column kk + ac
  const int br = lane & 3, bc = wn * WN + (lane >> 2);   // B frag: row kk + br, columns bc + 8 j
  const int sw = lane >> 2;                              // = (A frag row) & 7
  for (int it = 0; it < nk; ++it) {
    const int s = it % STAGES;
    mbar_wait(&full[s], (it / STAGES) & 1);
    const unsigned char* st = ring + s * T::STAGE_BYTES;
    const unsigned char* bs = st + T::A_BOXES * T::A_BOX_BYTES;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double a[C::MI], b[C::NI];
      const int ca = (kk & 15) + ac;                                   // column within the A box
      const unsigned char* abox = st + (kk >> 4) * T::A_BOX_BYTES;
#pragma unroll
      for (int i = 0; i < C::MI; ++i)
        a[i] = *reinterpret_cast<const double*>(abox + (ar + 8 * i) * 128 + ((((ca >> 1) ^ sw)) << 4) + (ca & 1) * 8);
      const int rb = kk + br, rsw = rb & 7;
#pragma unroll
      for (int j = 0; j < C::NI; ++j) {
        const int cb = bc + 8 * j, cc = cb & 15;
        b[j] = *reinterpret_cast<const double*>(bs + (cb >> 4) * T::B_BOX_BYTES + rb * 128 + (((cc >> 1) ^ rsw) << 4) +
                                                (cc & 1) * 8);
      }
#pragma unroll
      for (int i = 0; i < C::MI; ++i)
#pragma unroll
        for (int j = 0; j < C::NI; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);   // this warp is done with stage s
  }
  // epilogue (as gemm_ax_kernel): fragment (i, j) -> rows m0 + wm WM + 8 i + lane / 4,
  // cols wn WN + 8 j + 2 (lane % 4) + {0, 1}; k is even on this path
#pragma unroll
  for (int i = 0; i < C::MI; ++i) {
    const int64_t r = m0 + wm * WM + i * 8 + (lane >> 2);
    if (r >= M) continue;
#pragma unroll
    for (int j = 0; j < C::NI; ++j) {
      const int c = wn * WN + j * 8 + 2 * (lane & 3);
      if (c < k) *reinterpret_cast<double2*>(out + r * k + c) = make_double2(acc[i][j][0], acc[i][j][1]);
    }
  }
  if (fin.on) {   // consumer warps only (the producer has returned); every stage has been consumed
    __shared__ int s_last;
    fused_finish<C::THREADS, BM>(fin, (int)gridDim.x, out_split_stride, m0, tid, ring, &s_last,
                                 [] { asm volatile("bar.sync 1, %0;\n" ::"n"(C::THREADS) : "memory"); });
  }
}
template <int NT, int BM, int BK, int STAGES>
constexpr int gemm_tma_smem() { return STAGES * GemmTmaCfg<NT, BM, BK>::STAGE_BYTES + 1024 + 2 * STAGES * 8; }

__global__ void __launch_bounds__(256) w_finish_kernel(Ws ws, const double* __restrict__ X, int nsplit,
                                                      int64_t split_stride) {
  __shared__ dd sa[256], sg[256];
  griddep_wait();   // (programmatic dependent launch: the predecessor's writes are visible after this)
  if (*ws.status != ST_OK) return;
  const int64_t rows_per = (ws.n_loc + gridDim.x - 1) / gridDim.x;
  const int64_t rb = (int64_t)blockIdx.x * rows_per;
  const int64_t re = (rb + rows_per < ws.n_loc) ? rb + rows_per : ws.n_loc;
  tile_finish<256>(ws, X, nsplit, split_stride, rb, re, blockIdx.x, threadIdx.x, sa, sg);
  __syncthreads();
  tile_finish_slot<256>(ws, blockIdx.x, threadIdx.x, sa, sg);
}

}  // namespace rf
