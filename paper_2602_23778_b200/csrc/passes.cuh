// passes.cuh -- the tall-skinny row passes of a sweep over rows i >= top (rows below the
// k x k top block), on the FP64 tensor cores.
//
// pass B (S4 reductions): R = W - X^ D on the fly (Alg. 4 line 5 operand),
//   [M_2 | G_2] = X^_2^T [R_2 | X^_2]   (k x 2k, reduction over rows)  and  rr_j = sum r_ij^2.
//   A CTA owns one TA x TB output tile and one contiguous row chunk; partials go to fixed
//   slots and are summed in chunk order by passB_reduce (deterministic).  Per row it reads
//   x_i and w_i once (16 k bytes) for 2 k^2 FMAs.
// pass C (S6 update): x~_i = (w_i Sigma D^{-1}) - x^_i Csig   (the lower block of
//   X^ + H E_L, Alg. 4 line 7, via the identity in kxk.cuh), written to the X~ buffer (not in
//   place: CTAs of other column blocks still read the x^_i rows), plus column sums of x~^2 for
//   the normalisation.  Persistent CTAs keep a column block of Csig in shared memory.
// normalize (S7): x_ij = x~_ij / ||x~_j||, X~ buffer -> X.
#pragma once
#include <cuda.h>   // CUtensorMap

#include "common.cuh"

namespace rf {

constexpr int PB_RED_THREADS = 512;   // pass-B partial reduction: 32 elements x 16 chunk ranges per block

template <int KP, int TA, int TB, int WARPS_A, int WARPS_B, int BR>
struct PassBCfg {
  static constexpr int THREADS = WARPS_A * WARPS_B * 32;
  static constexpr int LDS = KP + ((KP % 16 == 8) ? 0 : 8);
  static constexpr int STAGE = BR * LDS;
  static constexpr int SMEM = 2 * 2 * STAGE * 8;       // X and W, double buffered
  static constexpr int WTA = TA / WARPS_A, WTB = TB / WARPS_B;
  static constexpr int MI = WTA / 8, NI = WTB / 8;
  static constexpr int NTA = KP / TA, NTB = 2 * KP / TB;
  // G = X^T X is symmetric: tiles of the G half lying strictly below its diagonal are skipped
  // (the reduction mirrors them), so tile ids enumerate only the kept (ta, tb) pairs.
  static constexpr __host__ __device__ bool kept(int ta, int tb) {
    return !(tb * TB >= KP && (tb * TB - KP) + TB <= ta * TA);
  }
  static constexpr __host__ __device__ int count() {
    int n = 0;
    for (int a = 0; a < NTA; ++a)
      for (int b = 0; b < NTB; ++b) n += kept(a, b) ? 1 : 0;
    return n;
  }
  static constexpr int NTILES = count();
  static __host__ __device__ int tile_id(int ta, int tb) {   // -1 if skipped
    int n = 0;
    for (int a = 0; a < NTA; ++a)
      for (int b = 0; b < NTB; ++b) {
        if (!kept(a, b)) continue;
        if (a == ta && b == tb) return n;
        ++n;
      }
    return -1;
  }
};

// R = W - X D is formed in place in the staged W rows for this tile's R columns (one fma per
// element, once per CTA), so the MMA loop reads one shared operand per fragment.  The tiles of
// the first a-block cover every R column exactly once; they also accumulate rr_j = sum r_ij^2.
template <int KP, int TA, int TB, int WARPS_A, int WARPS_B, int BR>
__global__ void __launch_bounds__(PassBCfg<KP, TA, TB, WARPS_A, WARPS_B, BR>::THREADS)
passB_kernel(Ws ws, const double* __restrict__ X, int vec16) {
  using C = PassBCfg<KP, TA, TB, WARPS_A, WARPS_B, BR>;
  constexpr int THREADS = C::THREADS;
  extern __shared__ __align__(16) double smem[];
  __shared__ double sd[KP];
  __shared__ double srr[THREADS];
  griddep_wait();   // (programmatic dependent launch: the predecessor's writes are visible after this)
  if (*ws.status != ST_OK) return;
  const int k = ws.k, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wa = warp / WARPS_B, wb = warp % WARPS_B;
  int ta = 0, tb = 0;
  {   // decode the kept-tile index
    int n = 0;
    for (int a = 0; a < C::NTA; ++a)
      for (int b = 0; b < C::NTB; ++b) {
        if (!C::kept(a, b)) continue;
        if (n == (int)blockIdx.x) { ta = a; tb = b; }
        ++n;
      }
  }
  const int a0 = ta * TA, b0 = tb * TB;
  const int rw = (b0 < KP) ? min(TB, KP - b0) : 0;      // R columns [b0, b0 + rw) of this tile
  const int64_t rows = ws.n_loc - ws.top;
  const int64_t per = ((rows + gridDim.y - 1) / gridDim.y + BR - 1) / BR * BR;
  const int64_t rb = ws.top + (int64_t)blockIdx.y * per;
  const int64_t re = (rb + per < ws.n_loc) ? rb + per : ws.n_loc;
  const int nit = (re > rb) ? (int)((re - rb + BR - 1) / BR) : 0;
  for (int j = tid; j < KP; j += THREADS) sd[j] = (j < k) ? ws.d[j] : 0.0;
  double* Xs = smem;
  double* Ws_ = smem + 2 * C::STAGE;

  auto load = [&](int buf, int it) {
    const int64_t r0 = rb + (int64_t)it * BR;
    double* xs = Xs + buf * C::STAGE;
    double* wsb = Ws_ + buf * C::STAGE;
    if (vec16) {
      for (int c = tid; c < BR * KP / 2; c += THREADS) {
        const int r = c / (KP / 2), cc = (c % (KP / 2)) * 2;
        const int64_t g = r0 + r;
        const bool ok = (g < re) && (cc < k);
        const int64_t off = ok ? g * k + cc : 0;
        cp_async16(xs + r * C::LDS + cc, X + off, ok);
        if (cc >= b0 && cc < b0 + rw) cp_async16(wsb + r * C::LDS + cc, ws.W + off, ok);
      }
    } else {
      for (int c = tid; c < BR * KP; c += THREADS) {
        const int r = c / KP, cc = c % KP;
        const int64_t g = r0 + r;
        const bool ok = (g < re) && (cc < k);
        const int64_t off = ok ? g * k + cc : 0;
        cp_async8(xs + r * C::LDS + cc, X + off, ok);
        if (cc >= b0 && cc < b0 + rw) cp_async8(wsb + r * C::LDS + cc, ws.W + off, ok);
      }
    }
  };

  double acc[C::MI][C::NI][2];
#pragma unroll
  for (int i = 0; i < C::MI; ++i)
#pragma unroll
    for (int j = 0; j < C::NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  double rr = 0.0;                                        // column b0 + tid % rw
  const bool do_rr = (ta == 0) && (rw > 0);
  if (nit > 0) load(0, 0);
  cp_async_commit();
  for (int it = 0; it < nit; ++it) {
    const int cur = it & 1;
    cp_async_wait<0>();
    __syncthreads();
    if (it + 1 < nit) load(cur ^ 1, it + 1);
    cp_async_commit();
    const double* xs = Xs + cur * C::STAGE;
    double* wsb = Ws_ + cur * C::STAGE;
    if (rw > 0) {
      for (int e = tid; e < BR * rw; e += THREADS) {     // R = W - X D  (fma as in the oracle)
        const int r = e / rw, c = b0 + e % rw;
        const double v = __fma_rn(-xs[r * C::LDS + c], sd[c], wsb[r * C::LDS + c]);
        wsb[r * C::LDS + c] = v;
        if (do_rr) rr = __fma_rn(v, v, rr);
      }
      __syncthreads();
    }
#pragma unroll
    for (int kk = 0; kk < BR; kk += 4) {
      const int row = kk + (lane & 3);
      double a[C::MI], b[C::NI];
#pragma unroll
      for (int i = 0; i < C::MI; ++i) a[i] = xs[row * C::LDS + a0 + wa * C::WTA + i * 8 + (lane >> 2)];
#pragma unroll
      for (int j = 0; j < C::NI; ++j) {
        const int cb8 = b0 + wb * C::WTB + j * 8;          // 8-column block: all R or all X (warp-uniform)
        const int col = cb8 + (lane >> 2);
        b[j] = (cb8 < KP) ? wsb[row * C::LDS + col] : xs[row * C::LDS + col - KP];
      }
#pragma unroll
      for (int i = 0; i < C::MI; ++i)
#pragma unroll
        for (int j = 0; j < C::NI; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
  }
  double* out = ws.bpart + ((int64_t)blockIdx.y * C::NTILES + blockIdx.x) * (TA * TB);
#pragma unroll
  for (int i = 0; i < C::MI; ++i)
#pragma unroll
    for (int j = 0; j < C::NI; ++j) {
      const int ra = wa * C::WTA + i * 8 + (lane >> 2);
      const int cb = wb * C::WTB + j * 8 + 2 * (lane & 3);
      out[ra * TB + cb] = acc[i][j][0];
      out[ra * TB + cb + 1] = acc[i][j][1];
    }
  if (do_rr) {   // threads t, t + rw, ... share column b0 + t % rw (THREADS is a multiple of rw)
    srr[tid] = rr;
    __syncthreads();
    if (tid < rw) {
      double sum = srr[tid];
      for (int q = 1; q < THREADS / rw; ++q) sum += srr[q * rw + tid];
      ws.brr[(int64_t)blockIdx.y * KP + b0 + tid] = sum;
    }
  }
}

// sum_{c < n} p[c * stride] in ascending c (loads batched 8 at a time so they overlap)
__device__ __forceinline__ double sum_strided(const double* __restrict__ p, int64_t stride, int n) {
  double s = 0.0;
  int c = 0;
  for (; c + 8 <= n; c += 8) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = p[(int64_t)(c + u) * stride];
#pragma unroll
    for (int u = 0; u < 8; ++u) s += v[u];
  }
  for (; c < n; ++c) s += p[(int64_t)c * stride];
  return s;
}

// Sum pass-B partials over chunks in fixed order -> M2 (k x k), G2 (k x k), rr2 (k).
// Block = 32 elements x NR contiguous chunk ranges; the NR range sums are combined in order.
template <int KP, int TA, int TB, int WARPS_A, int WARPS_B, int BR>
__global__ void __launch_bounds__(PB_RED_THREADS) passB_reduce_kernel(Ws ws, int nchunk) {
  using C = PassBCfg<KP, TA, TB, WARPS_A, WARPS_B, BR>;
  constexpr int NR = PB_RED_THREADS / 32;              // contiguous chunk ranges per element
  __shared__ double part[NR][33];
  griddep_wait();   // (programmatic dependent launch: the predecessor's writes are visible after this)
  if (*ws.status != ST_OK) return;
  const int k = ws.k;
  const int total = k * 2 * k + k;
  const int el = threadIdx.x & 31, rg = threadIdx.x >> 5;
  const int e = blockIdx.x * 32 + el;
  const int c0 = (int)((int64_t)nchunk * rg / NR), c1 = (int)((int64_t)nchunk * (rg + 1) / NR);
  double s = 0.0;
  if (e < total) {
    if (e >= 2 * k * k) {
      const int j = e - 2 * k * k;
      s = sum_strided(ws.brr + (int64_t)c0 * KP + j, KP, c1 - c0);
    } else {
      int a = e / (2 * k), bb = e % (2 * k);
      if (bb >= k) {                                   // G half: mirror skipped (lower) tiles
        const int gb = bb - k;
        if (C::tile_id(a / TA, (KP + gb) / TB) < 0) { const int t = a; a = gb; bb = k + t; }
      }
      const int b = (bb < k) ? bb : KP + (bb - k);     // column in the padded [R | X] space
      const int tile = C::tile_id(a / TA, b / TB);
      const int off = (a % TA) * TB + (b % TB);
      s = sum_strided(ws.bpart + ((int64_t)c0 * C::NTILES + tile) * (TA * TB) + off,
                      (int64_t)C::NTILES * TA * TB, c1 - c0);
    }
  }
  part[rg][el] = s;
  __syncthreads();
  if (rg == 0 && e < total) {
    for (int q = 1; q < NR; ++q) s += part[q][el];
    if (e >= 2 * k * k) {
      ws.rr2[e - 2 * k * k] = s;
    } else {
      const int a = e / (2 * k), bb = e % (2 * k);
      if (bb < k) ws.M2[a * k + bb] = s;
      else ws.G2[a * k + (bb - k)] = s;
    }
  }
}

// ---------------------------------------------------------------- pass B, k >= 32
// CTA tile = all KP output rows a (the X^ columns) x one 64-wide block tb of the [R | X^] column
// space, so every staged row is read by the CTA's MMAs TA x 64 / (KP + R width) times and the
// CTA count per row chunk is 2 KP / 64.  BR = 32 rows per stage, one barrier per stage (8 k-steps
// of DMMA).  The symmetric G half: warp tiles lying strictly below G's diagonal issue no MMAs (the
// reduction mirrors them), so no flops are spent on them.  R = W - X D is formed in place in the
// staged W columns of R tiles (one fma per element, exactly once per element over the grid) by
// the thread that copied both operands, right after its own copies of the NEXT stage land --
// so the R formation needs no barrier of its own and overlaps the other warps' MMAs; the R tiles
// also accumulate rr_j = sum r_ij^2.
template <int KP, int WA_ = 2, int WB_ = 4, int BR_ = 32>
struct PassB2Cfg {
  static constexpr int TA = KP, TB = 64, NT = 2 * KP / TB;
  static constexpr int WA = WA_, WB = WB_;                     // default 8 warps
  static constexpr int THREADS = WA * WB * 32;
  static constexpr int WTA = TA / WA, WTB = TB / WB;           // warp tile (KP=128: 64 x 16)
  static constexpr int MI = WTA / 8, NI = WTB / 8;
  static constexpr int BR = BR_;
  static constexpr int LDX = KP + ((KP % 16 == 8) ? 0 : 8);
  static constexpr int LDW = (KP < TB ? KP : TB) + 8;          // staged R columns of a tile
  static constexpr int XST = BR * LDX, WST = BR * LDW;
  static constexpr int SMEM = 2 * (XST + WST) * 8;
  static constexpr bool PAIRED = (KP == 128 && WA == 2);       // balanced 7-unit grid (see passB2_kernel)
  static constexpr int MINB = (2 * (XST + WST) * 8 <= 113 * 1024) ? 2 : 1;   // 2 CTAs / SM when smem allows
};

template <int KP, int WA_ = 2, int WB_ = 4, int BR_ = 32>
__global__ void __launch_bounds__(PassB2Cfg<KP, WA_, WB_, BR_>::THREADS, PassB2Cfg<KP, WA_, WB_, BR_>::MINB)
passB2_kernel(Ws ws, const double* __restrict__ X, int vec16) {
  using C = PassB2Cfg<KP, WA_, WB_, BR_>;
  constexpr int THREADS = C::THREADS, BR = C::BR, TB = C::TB;
  extern __shared__ __align__(16) double smem[];
  __shared__ double sd[KP];
  __shared__ double srr[2][THREADS];
  griddep_wait();   // (programmatic dependent launch: the predecessor's writes are visible after this)
  if (*ws.status != ST_OK) return;
  const int k = ws.k, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wa = warp / C::WB, wb = warp % C::WB;
  // KP = 128: the X0 tile does half the MMAs of the others (G10 skipped), so the grid is made of
  // balanced work units -- per pair of row chunks: R0, R1, X1 for each chunk (6 units) plus one
  // X0 unit spanning both chunks (gridDim.x = 7 x pairs).  Otherwise gridDim = (NT, chunks).
  int tb, span = 1;
  int64_t cidx, nchunk;
  if (C::PAIRED) {
    const int u = blockIdx.x, pair = u / 7, w = u % 7;
    nchunk = 2 * (int64_t)(gridDim.x / 7);
    if (w < 6) { tb = (w % 3 == 2) ? 3 : (w % 3); cidx = 2 * pair + w / 3; }
    else { tb = 2; cidx = 2 * pair; span = 2; }
  } else {
    tb = blockIdx.x; cidx = blockIdx.y; nchunk = gridDim.y;
  }
  const int b0 = tb * TB;                                     // [R | X] columns [b0, b0 + 64)
  const int rw = (b0 < KP) ? min(TB, KP - b0) : 0;           // R columns of this tile: [b0, b0 + rw)
  const int64_t rows = ws.n_loc - ws.top;
  const int64_t per = ((rows + nchunk - 1) / nchunk + BR - 1) / BR * BR;
  const int64_t rb = ws.top + cidx * per;
  const int64_t re = (rb + span * per < ws.n_loc) ? rb + span * per : ws.n_loc;
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
        cp_async16(wsb + r * C::LDW + cc, ws.W + (ok ? g * k + b0 + cc : 0), ok);
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
      rr0 = __fma_rn(v0, v0, rr0);
      if (rpair == 2) {
        const double v1 = __fma_rn(-xs[r * C::LDX + b0 + rcol + 1], d1, wsb[r * C::LDW + rcol + 1]);
        wsb[r * C::LDW + rcol + 1] = v1;
        rr1 = __fma_rn(v1, v1, rr1);
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
    if (it + 1 < nit) load(cur ^ 1, it + 1);
    cp_async_commit();
    const double* xs = Xs + cur * C::XST;
    const double* wsb = Wsm + cur * C::WST;
    if (active) {
#pragma unroll
      for (int kk = 0; kk < BR; kk += 4) {
        const int row = kk + (lane & 3);
        double a[C::MI], b[C::NI];
#pragma unroll
        for (int i = 0; i < C::MI; ++i) a[i] = xs[row * C::LDX + a_lo + i * 8 + (lane >> 2)];
#pragma unroll
        for (int j = 0; j < C::NI; ++j) {
          const int cb8 = bw + j * 8;                         // 8-column block: all R or all X (warp-uniform)
          b[j] = (cb8 < KP) ? wsb[row * C::LDW + (cb8 - b0) + (lane >> 2)] : xs[row * C::LDX + cb8 - KP + (lane >> 2)];
        }
#pragma unroll
        for (int i = 0; i < C::MI; ++i)
#pragma unroll
          for (int j = 0; j < C::NI; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
      }
    }
    cp_async_wait<0>();
    if (rw > 0 && it + 1 < nit) form_r(cur ^ 1);
  }
  if (active) {
    for (int q = 0; q < span; ++q) {          // a two-chunk unit stores its sum in the first slot, 0 in the second
      double* out = ws.bpart + ((cidx + q) * C::NT + tb) * (C::TA * TB);
#pragma unroll
      for (int i = 0; i < C::MI; ++i)
#pragma unroll
        for (int j = 0; j < C::NI; ++j) {
          const int ra = a_lo + i * 8 + (lane >> 2);
          const int cb = wb * C::WTB + j * 8 + 2 * (lane & 3);
          out[ra * TB + cb] = q ? 0.0 : acc[i][j][0];
          out[ra * TB + cb + 1] = q ? 0.0 : acc[i][j][1];
        }
    }
  }
  if (rw > 0) {   // threads t, t + rcpr, ... share the R column(s) b0 + rcol (+1): fixed-order sum
    srr[0][tid] = rr0;
    srr[1][tid] = rr1;
    __syncthreads();
    if (tid < rcpr) {
      double s0 = srr[0][tid], s1 = srr[1][tid];
      for (int q = 1; q < THREADS / rcpr; ++q) { s0 += srr[0][q * rcpr + tid]; s1 += srr[1][q * rcpr + tid]; }
      ws.brr[cidx * KP + b0 + rcol] = s0;
      if (rpair == 2) ws.brr[cidx * KP + b0 + rcol + 1] = s1;
    }
  }
}

// ---------------------------------------------------------------- pass B at k = 128, fed by TMA
// Same units (7 per pair of row chunks), warp tiles, skipped G warp tiles and partial-slot layout as
// passB2_kernel, but the X^ and W slabs of each 16-row stage arrive as 128-byte-swizzled 2-D TMA boxes
// (16 doubles wide) issued by one producer warp into a 4-stage full / empty mbarrier ring (the dense
// GEMM's scheme, gemm_dense.cuh): no per-thread copies in the main loop.  R = W - X D is formed in
// place in the W boxes by the consumer threads (thread t always owns column t % 64 -> its share of
// rr_j), then a named barrier among the consumers, then the DMMAs.
template <int KP>
struct PassB2TmaCfg {
  static constexpr int TA = KP, TB = 64, NT = 2 * KP / TB;
  static constexpr int WA = 2, WB = 4, WARPS = WA * WB, THREADS = WARPS * 32;
  static constexpr int WTA = TA / WA, WTB = TB / WB, MI = WTA / 8, NI = WTB / 8;
  static constexpr int BR = 32, ST = 4;
  static constexpr int XBOXES = KP / 16, WBOXES = TB / 16, BOX = BR * 128;
  static constexpr int STAGE = (XBOXES + WBOXES) * BOX;
  static constexpr int SMEM = ST * STAGE + 1024 + 2 * ST * 8;
};
// byte offset of element (r, c) in an array of 16-column swizzled boxes of BR rows
template <int BR>
RF_DEV int swz_off(int r, int c) {
  return (c >> 4) * (BR * 128) + r * 128 + ((((c & 15) >> 1) ^ (r & 7)) << 4) + (c & 1) * 8;
}
template <int KP>
__global__ void __launch_bounds__(PassB2TmaCfg<KP>::THREADS + 32, 1)
passB2_tma_kernel(Ws ws, const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW) {
  using C = PassB2TmaCfg<KP>;
  constexpr int BR = C::BR, TB = C::TB, ST = C::ST;
  extern __shared__ __align__(1024) unsigned char pbsm[];
  __shared__ double sd[KP];
  __shared__ double srr[C::THREADS];
  griddep_wait();
  if (*ws.status != ST_OK) return;
  unsigned char* ring = smem_align1024(pbsm);
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + ST * C::STAGE);
  uint64_t* empty = full + ST;
  const int k = ws.k, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // units: per pair of row chunks R0, R1, X1 for each chunk plus one X0 unit spanning both
  const int u = blockIdx.x, pair = u / 7, w7 = u % 7;
  const int64_t nchunk = 2 * (int64_t)(gridDim.x / 7);
  int tb, span = 1;
  int64_t cidx;
  if (w7 < 6) { tb = (w7 % 3 == 2) ? 3 : (w7 % 3); cidx = 2 * pair + w7 / 3; }
  else { tb = 2; cidx = 2 * pair; span = 2; }
  const int b0 = tb * TB;
  const int rw = (b0 < KP) ? min(TB, KP - b0) : 0;           // R columns of this tile
  const int64_t rows = ws.n_loc - ws.top;
  const int64_t per = ((rows + nchunk - 1) / nchunk + 31) / 32 * 32;   // (passB2's chunking; a multiple of BR)
  const int64_t rb = ws.top + cidx * per;
  const int64_t re = (rb + span * per < ws.n_loc) ? rb + span * per : ws.n_loc;
  const int nit = (re > rb) ? (int)((re - rb + BR - 1) / BR) : 0;
  for (int j = tid; j < KP; j += blockDim.x) sd[j] = (j < k) ? ws.d[j] : 0.0;
  if (tid == 0) {
    for (int s = 0; s < ST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], C::WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (warp == C::WARPS) {   // producer warp
    if (lane == 0) {
      const uint32_t bytes = (C::XBOXES + (rw > 0 ? C::WBOXES : 0)) * C::BOX;
      for (int it = 0; it < nit; ++it) {
        const int s = it % ST;
        if (it >= ST) {
          mbar_wait(&empty[s], ((it / ST) - 1) & 1);
          fence_async_smem();                     // consumers' generic reads / R writes of stage s -> refill
        }
        unsigned char* st = ring + s * C::STAGE;
        const int r0 = (int)(rb + (int64_t)it * BR);
        mbar_expect_tx(&full[s], bytes);
#pragma unroll
        for (int b = 0; b < C::XBOXES; ++b) tma_load_2d(st + b * C::BOX, &tmX, 16 * b, r0, &full[s]);
        if (rw > 0) {
#pragma unroll
          for (int b = 0; b < C::WBOXES; ++b)
            tma_load_2d(st + (C::XBOXES + b) * C::BOX, &tmW, b0 + 16 * b, r0, &full[s]);
        }
      }
    }
    return;
  }
  const int wa = warp / C::WB, wb = warp % C::WB;
  const int a_lo = wa * C::WTA, bw = b0 + wb * C::WTB;
  const bool active = !(bw >= KP && a_lo >= (bw - KP) + C::WTB);   // below G's diagonal: no MMAs
  const int rcol = tid % TB;                                        // this thread's R column b0 + rcol
  const double drc = sd[b0 + rcol < KP ? b0 + rcol : 0];
  double rr = 0.0;
  double acc[C::MI][C::NI][2];
#pragma unroll
  for (int i = 0; i < C::MI; ++i)
#pragma unroll
    for (int j = 0; j < C::NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  for (int it = 0; it < nit; ++it) {
    const int s = it % ST;
    mbar_wait(&full[s], (it / ST) & 1);
    const unsigned char* xs = ring + s * C::STAGE;
    unsigned char* wsb = ring + s * C::STAGE + C::XBOXES * C::BOX;
    if (rw > 0) {   // R = W - X D in place (rows beyond the matrix are zero-filled: R = 0)
#pragma unroll
      for (int q = 0; q < BR * TB / C::THREADS; ++q) {
        const int r = tid / TB + q * (C::THREADS / TB);
        double* wp = reinterpret_cast<double*>(wsb + swz_off<BR>(r, rcol));
        const double x = *reinterpret_cast<const double*>(xs + swz_off<BR>(r, b0 + rcol));
        const double v = __fma_rn(-x, drc, *wp);
        *wp = v;
        rr = __fma_rn(v, v, rr);
      }
      asm volatile("bar.sync 1, %0;\n" ::"n"(C::THREADS) : "memory");   // consumers only
    }
    if (active) {
#pragma unroll
      for (int kk = 0; kk < BR; kk += 4) {
        // the 4 k rows of this DMMA step: {8 (kk / 8) + (kk / 4) % 2 + 2 t}, t = lane & 3 -- rows whose
        // r % 8 differ by 2, so with the 128-byte swizzle the 4 rows x 4 columns of a half-warp hit 8
        // distinct 16-byte chunks (adjacent rows kk + t mapped 2 rows onto the same chunks: 2-way
        // bank conflicts on every fragment load)
        const int row = (kk & ~7) + ((kk >> 2) & 1) + 2 * (lane & 3);
        double a[C::MI], bv[C::NI];
#pragma unroll
        for (int i = 0; i < C::MI; ++i)
          a[i] = *reinterpret_cast<const double*>(xs + swz_off<BR>(row, a_lo + i * 8 + (lane >> 2)));
#pragma unroll
        for (int j = 0; j < C::NI; ++j) {
          const int cb8 = bw + j * 8;                                 // all R or all X (warp-uniform)
          bv[j] = (cb8 < KP) ? *reinterpret_cast<const double*>(wsb + swz_off<BR>(row, cb8 - b0 + (lane >> 2)))
                             : *reinterpret_cast<const double*>(xs + swz_off<BR>(row, cb8 - KP + (lane >> 2)));
        }
#pragma unroll
        for (int i = 0; i < C::MI; ++i)
#pragma unroll
          for (int j = 0; j < C::NI; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], bv[j]);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
  if (active) {
    for (int q = 0; q < span; ++q) {          // a two-chunk unit stores its sum in the first slot, 0 in the second
      double* out = ws.bpart + ((cidx + q) * C::NT + tb) * (C::TA * TB);
#pragma unroll
      for (int i = 0; i < C::MI; ++i)
#pragma unroll
        for (int j = 0; j < C::NI; ++j) {
          const int ra = a_lo + i * 8 + (lane >> 2);
          const int cb = wb * C::WTB + j * 8 + 2 * (lane & 3);
          out[ra * TB + cb] = q ? 0.0 : acc[i][j][0];
          out[ra * TB + cb + 1] = q ? 0.0 : acc[i][j][1];
        }
    }
  }
  if (rw > 0) {   // threads rcol, rcol + 64, ... share R column b0 + rcol: fixed-order sum
    srr[tid] = rr;
    asm volatile("bar.sync 1, %0;\n" ::"n"(C::THREADS) : "memory");
    if (tid < TB && b0 + tid < KP) {
      double sacc = srr[tid];
      for (int q = 1; q < C::THREADS / TB; ++q) sacc += srr[q * TB + tid];
      ws.brr[cidx * KP + b0 + tid] = sacc;
    }
  }
}

// ---------------------------------------------------------------- pass B at k = 128, ping-pong
// passB2_tma_kernel's units, ring and slot layout, but the CTA's 64 tile columns are split between
// two consumer groups of 8 warps (32 columns each, 4 x 2 warp tiles of 32 x 16).  Each group forms
// R for its own columns and meets at its own named barrier, so while one group forms R the other
// can issue DMMAs, and the groups drift apart instead of idling the DMMA pipe together at every
// stage.  No producer warp (16 warps keep 128 registers): the last of the 16 warps through a stage
// refills it.  Same per-element DMMA k-order as passB2_tma_kernel (identical partials); rr_j is
// summed over the 8 threads of a column in a fixed order.
struct PassB2PPCfg {
  static constexpr int KP = 128, TA = KP, TB = 64, NT = 2 * KP / TB;
  static constexpr int GROUPS = 2, GWARPS = 8, WARPS = GROUPS * GWARPS, THREADS = WARPS * 32, GTHREADS = GWARPS * 32;
  static constexpr int GCOLS = TB / GROUPS, WA = 4, WB = 2;
  static constexpr int WTA = TA / WA, WTB = GCOLS / WB, MI = WTA / 8, NI = WTB / 8;
  static constexpr int BR = 32, ST = 4;
  static constexpr int XBOXES = KP / 16, WBOXES = TB / 16, BOX = BR * 128;
  static constexpr int STAGE = (XBOXES + WBOXES) * BOX;
  static constexpr int SMEM = ST * STAGE + 1024 + ST * 8 + ST * 4;
};
__global__ void __launch_bounds__(PassB2PPCfg::THREADS, 1)
passB2_pp_kernel(Ws ws, const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW) {
  using C = PassB2PPCfg;
  constexpr int BR = C::BR, TB = C::TB, ST = C::ST, KP = C::KP;
  extern __shared__ __align__(1024) unsigned char pbsm[];
  __shared__ double sd[KP];
  __shared__ double srr[C::THREADS];
  griddep_wait();
  if (*ws.status != ST_OK) return;
  unsigned char* ring = smem_align1024(pbsm);
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + ST * C::STAGE);
  int* done = reinterpret_cast<int*>(full + ST);                    // warps through a stage (monotonic)
  const int k = ws.k, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // units: per pair of row chunks R0, R1, X1 for each chunk plus one X0 unit spanning both
  const int u = blockIdx.x, pair = u / 7, w7 = u % 7;
  const int64_t nchunk = 2 * (int64_t)(gridDim.x / 7);
  int tb, span = 1;
  int64_t cidx;
  if (w7 < 6) { tb = (w7 % 3 == 2) ? 3 : (w7 % 3); cidx = 2 * pair + w7 / 3; }
  else { tb = 2; cidx = 2 * pair; span = 2; }
  const int b0 = tb * TB;
  const bool rtile = b0 < KP;                                 // all 64 columns are R columns (else X)
  const int64_t rows = ws.n_loc - ws.top;
  const int64_t per = ((rows + nchunk - 1) / nchunk + 31) / 32 * 32;   // (passB2's chunking; a multiple of BR)
  const int64_t rb = ws.top + cidx * per;
  // stages of each of the unit's chunks (a two-chunk X0 unit interleaves them: stage s of chunk a, then
  // stage s of chunk b, so it reads the X^ rows its two chunks' other units read at the same time and
  // they stay in L2 for them -- reading chunk a then chunk b ran it twice as fast through each chunk as
  // its siblings, so its X^ rows came from DRAM twice)
  auto chunk_stages = [&](int64_t c0) -> int {
    const int64_t e = (c0 + per < ws.n_loc) ? c0 + per : ws.n_loc;
    return (e > c0) ? (int)((e - c0 + BR - 1) / BR) : 0;
  };
  const int nit_a = chunk_stages(rb), nit_b = (span == 2) ? chunk_stages(rb + per) : 0;
  const int nit = nit_a + nit_b, nmin = nit_a < nit_b ? nit_a : nit_b;
  auto stage_row = [&](int it) -> int64_t {
    if (span == 1) return rb + (int64_t)it * BR;
    if (it < 2 * nmin) return rb + (it & 1) * per + (int64_t)(it >> 1) * BR;
    return rb + (nit_a > nit_b ? 0 : per) + (int64_t)(nmin + it - 2 * nmin) * BR;
  };
  auto issue = [&](int it) {
    const int s = it % ST;
    unsigned char* st = ring + s * C::STAGE;
    const int r0 = (int)stage_row(it);
    mbar_expect_tx(&full[s], (C::XBOXES + (rtile ? C::WBOXES : 0)) * C::BOX);
#pragma unroll
    for (int b = 0; b < C::XBOXES; ++b) tma_load_2d(st + b * C::BOX, &tmX, 16 * b, r0, &full[s]);
    if (rtile) {
#pragma unroll
      for (int b = 0; b < C::WBOXES; ++b) tma_load_2d(st + (C::XBOXES + b) * C::BOX, &tmW, b0 + 16 * b, r0, &full[s]);
    }
  };
  for (int j = tid; j < KP; j += blockDim.x) sd[j] = (j < k) ? ws.d[j] : 0.0;
  if (tid == 0) {
    for (int s = 0; s < ST; ++s) { mbar_init(&full[s], 1); done[s] = 0; }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    for (int it = 0; it < ST && it < nit; ++it) issue(it);
  }
  __syncthreads();
  const int grp = warp / C::GWARPS, gw = warp % C::GWARPS, gtid = tid - grp * C::GTHREADS;
  const int wa = gw / C::WB, wb = gw % C::WB;
  const int a_lo = wa * C::WTA, bw = b0 + grp * C::GCOLS + wb * C::WTB;   // warp tile column (padded [R | X])
  const bool active = !(bw >= KP && a_lo >= (bw - KP) + C::WTB);          // below G's diagonal: no MMAs
  const int rcol = grp * C::GCOLS + gtid % C::GCOLS;                       // this thread's R column (in the tile)
  const double drc = rtile ? sd[b0 + rcol] : 0.0;
  double rr = 0.0;
  double acc[C::MI][C::NI][2];
#pragma unroll
  for (int i = 0; i < C::MI; ++i)
#pragma unroll
    for (int j = 0; j < C::NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  for (int it = 0; it < nit; ++it) {
    const int s = it % ST;
    mbar_wait(&full[s], (it / ST) & 1);
    const unsigned char* xs = ring + s * C::STAGE;
    unsigned char* wsb = ring + s * C::STAGE + C::XBOXES * C::BOX;
    if (rtile) {   // R = W - X D in place for this group's columns (zero-filled rows: R = 0)
#pragma unroll
      for (int q = 0; q < BR * C::GCOLS / C::GTHREADS; ++q) {
        const int r = gtid / C::GCOLS + q * (C::GTHREADS / C::GCOLS);
        double* wp = reinterpret_cast<double*>(wsb + swz_off<BR>(r, rcol));
        const double x = *reinterpret_cast<const double*>(xs + swz_off<BR>(r, b0 + rcol));
        const double v = __fma_rn(-x, drc, *wp);
        *wp = v;
        rr = __fma_rn(v, v, rr);
      }
      asm volatile("bar.sync %0, %1;\n" ::"r"(1 + grp), "n"(C::GTHREADS) : "memory");   // this group only
    }
    if (active) {
#pragma unroll
      for (int kk = 0; kk < BR; kk += 4) {
        // the 4 k rows of this DMMA step: {8 (kk / 8) + (kk / 4) % 2 + 2 t}, t = lane & 3 -- rows whose
        // r % 8 differ by 2, so with the 128-byte swizzle the 4 rows x 4 columns of a half-warp hit 8
        // distinct 16-byte chunks (adjacent rows kk + t mapped 2 rows onto the same chunks: 2-way
        // bank conflicts on every fragment load)
        const int row = (kk & ~7) + ((kk >> 2) & 1) + 2 * (lane & 3);
        double a[C::MI], bv[C::NI];
#pragma unroll
        for (int i = 0; i < C::MI; ++i)
          a[i] = *reinterpret_cast<const double*>(xs + swz_off<BR>(row, a_lo + i * 8 + (lane >> 2)));
#pragma unroll
        for (int j = 0; j < C::NI; ++j) {
          const int cb8 = bw + j * 8;                                 // all R or all X (warp-uniform)
          bv[j] = (cb8 < KP) ? *reinterpret_cast<const double*>(wsb + swz_off<BR>(row, cb8 - b0 + (lane >> 2)))
                             : *reinterpret_cast<const double*>(xs + swz_off<BR>(row, cb8 - KP + (lane >> 2)));
        }
#pragma unroll
        for (int i = 0; i < C::MI; ++i)
#pragma unroll
          for (int j = 0; j < C::NI; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], bv[j]);
      }
    }
    __syncwarp();                                // this warp's reads / R writes of the stage are done
    if (lane == 0 && stage_release_last(&done[s], C::WARPS) && it + ST < nit) issue(it + ST);   // last of the 16 warps: refill
  }
  if (active) {
    for (int q = 0; q < span; ++q) {          // a two-chunk unit stores its sum in the first slot, 0 in the second
      double* out = ws.bpart + ((cidx + q) * C::NT + tb) * (C::TA * TB);
#pragma unroll
      for (int i = 0; i < C::MI; ++i)
#pragma unroll
        for (int j = 0; j < C::NI; ++j) {
          const int ra = a_lo + i * 8 + (lane >> 2);
          const int cb = (bw - b0) + j * 8 + 2 * (lane & 3);
          out[ra * TB + cb] = q ? 0.0 : acc[i][j][0];
          out[ra * TB + cb + 1] = q ? 0.0 : acc[i][j][1];
        }
    }
  }
  if (rtile) {   // the 8 threads of a column (gtid = c % 32 + 32 q within its group): fixed-order sum
    srr[tid] = rr;
    __syncthreads();
    if (tid < TB && b0 + tid < KP) {
      const int g = tid / C::GCOLS, cc = tid % C::GCOLS;
      double sacc = srr[g * C::GTHREADS + cc];
      for (int q = 1; q < C::GTHREADS / C::GCOLS; ++q) sacc += srr[g * C::GTHREADS + cc + q * C::GCOLS];
      ws.brr[cidx * KP + b0 + tid] = sacc;
    }
  }
}

// Sum pass-B2 partials over chunks in fixed order -> M2, G2 (mirrored from its upper triangle), rr2.
template <int KP>
__global__ void __launch_bounds__(PB_RED_THREADS) passB2_reduce_kernel(Ws ws, int nchunk) {
  using C = PassB2Cfg<KP>;
  constexpr int NR = PB_RED_THREADS / 32;              // contiguous chunk ranges per element
  __shared__ double part[NR][33];
  griddep_wait();   // (programmatic dependent launch: the predecessor's writes are visible after this)
  if (*ws.status != ST_OK) return;
  const int k = ws.k;
  const int total = k * 2 * k + k;
  const int el = threadIdx.x & 31, rg = threadIdx.x >> 5;
  const int e = blockIdx.x * 32 + el;
  const int c0 = (int)((int64_t)nchunk * rg / NR), c1 = (int)((int64_t)nchunk * (rg + 1) / NR);
  double s = 0.0;
  if (e < total) {
    if (e >= 2 * k * k) {
      const int j = e - 2 * k * k;
      s = sum_strided(ws.brr + (int64_t)c0 * KP + j, KP, c1 - c0);
    } else {
      int a = e / (2 * k), bb = e % (2 * k);
      if (ws.bdiag && (bb == a || bb == k + a)) {        // tcgen05 pass B: the FP64 diagonals
        s = sum_strided(ws.bdiag + (int64_t)c0 * 2 * KP + (bb == a ? 0 : KP) + a, 2 * KP, c1 - c0);
      } else {
        int col;                                         // column in the padded [R | X] space
        if (bb < k) {
          col = bb;
        } else {                                         // G[a][g] = G[min][max] (upper triangle)
          const int g = bb - k, lo = a < g ? a : g, hi = a < g ? g : a;
          a = lo;
          col = KP + hi;
        }
        const int tile = col / C::TB, off = a * C::TB + (col % C::TB);
        s = sum_strided(ws.bpart + ((int64_t)c0 * C::NT + tile) * (C::TA * C::TB) + off,
                        (int64_t)C::NT * C::TA * C::TB, c1 - c0);
      }
    }
  }
  part[rg][el] = s;
  __syncthreads();
  if (rg == 0 && e < total) {
    for (int q = 1; q < NR; ++q) s += part[q][el];
    if (e >= 2 * k * k) {
      ws.rr2[e - 2 * k * k] = s;
    } else {
      const int a = e / (2 * k), bb = e % (2 * k);
      if (bb < k) ws.M2[a * k + bb] = s;
      else ws.G2[a * k + (bb - k)] = s;
    }
  }
}

// pass C CTA: BM rows x NC output columns (blockIdx.y selects the column block), Csig[:, cols]
// resident in shared memory for the CTA's lifetime (persistent over row tiles).
template <int KP, int NC, int BM, int WARPS_M, int WARPS_N>
struct PassCCfg {
  static constexpr int THREADS = WARPS_M * WARPS_N * 32;
  static constexpr int LDX = KP + 4;                               // A-frag reads (8 rows x 4)
  static constexpr int LDC = NC + ((NC % 16 == 8) ? 0 : 8);        // B-frag reads (4 rows x 8)
  static constexpr int XSTAGE = BM * LDX;
  static constexpr int SMEM = (KP * LDC + 2 * XSTAGE) * 8;
  static constexpr int WM = BM / WARPS_M, WN = NC / WARPS_N;
  static constexpr int MI = WM / 8, NI = WN / 8;
};

// NORM: also the column sums of x~^2 into ws.nslot (Rayleigh-Ritz / QR steps, which normalise afterwards).
// A sweep's Csig and scal already carry 1 / ||x~_j|| (kxk_finish), so its pass C skips them: the two
// DFMA per element cost far more than their pipe share next to the DMMAs.
template <int KP, int NC, int BM, int WARPS_M, int WARPS_N, bool NORM = true>
__global__ void __launch_bounds__(PassCCfg<KP, NC, BM, WARPS_M, WARPS_N>::THREADS)
passC_kernel(Ws ws, const double* X, double* out, int vec16) {
  using C = PassCCfg<KP, NC, BM, WARPS_M, WARPS_N>;
  extern __shared__ __align__(16) double smem[];
  __shared__ double ssc[NC];
  __shared__ double sred[WARPS_M * 8][NC];
  griddep_wait();   // (programmatic dependent launch: the predecessor's writes are visible after this)
  if (*ws.status != ST_OK) return;
  const int k = ws.k, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / WARPS_N, wn = warp % WARPS_N;
  const int n0 = blockIdx.y * NC;                  // first output column of this CTA
  double* Cs = smem;
  double* Xs = smem + KP * C::LDC;
  for (int l = tid / NC; l < KP; l += C::THREADS / NC) {
    const int j = tid % NC;
    Cs[l * C::LDC + j] = (l < k && n0 + j < k) ? ws.Csig[l * k + n0 + j] : 0.0;
  }
  for (int j = tid; j < NC; j += C::THREADS) ssc[j] = (n0 + j < k) ? ws.scal[n0 + j] : 0.0;
  const int64_t rows = ws.n_loc - ws.top;
  const int64_t ntile = (rows + BM - 1) / BM;

  auto load = [&](int buf, int64_t t) {
    const int64_t r0 = ws.top + t * BM;
    double* xs = Xs + buf * C::XSTAGE;
    if (vec16) {
      for (int c = tid; c < BM * KP / 2; c += C::THREADS) {
        const int r = c / (KP / 2), cc = (c % (KP / 2)) * 2;
        const int64_t g = r0 + r;
        const bool ok = (g < ws.n_loc) && (cc < k);
        cp_async16(xs + r * C::LDX + cc, X + (ok ? g * k + cc : 0), ok);
      }
    } else {
      for (int c = tid; c < BM * KP; c += C::THREADS) {
        const int r = c / KP, cc = c % KP;
        const int64_t g = r0 + r;
        const bool ok = (g < ws.n_loc) && (cc < k);
        cp_async8(xs + r * C::LDX + cc, X + (ok ? g * k + cc : 0), ok);
      }
    }
  };

  double nacc[C::NI][2];
#pragma unroll
  for (int j = 0; j < C::NI; ++j) nacc[j][0] = nacc[j][1] = 0.0;
  int64_t t = blockIdx.x;
  if (t < ntile) load(0, t);
  cp_async_commit();
  for (int buf = 0; t < ntile; t += gridDim.x, buf ^= 1) {
    cp_async_wait<0>();
    __syncthreads();
    if (t + gridDim.x < ntile) load(buf ^ 1, t + gridDim.x);
    cp_async_commit();
    const int64_t r0 = ws.top + t * BM;
    // prefetch this thread's W entries (independent of the MMA loop)
    double w[C::MI][C::NI][2];
#pragma unroll
    for (int i = 0; i < C::MI; ++i) {
      const int64_t g = r0 + wm * C::WM + i * 8 + (lane >> 2);
#pragma unroll
      for (int j = 0; j < C::NI; ++j) {
        const int c = n0 + wn * C::WN + j * 8 + 2 * (lane & 3);
        const bool okr = g < ws.n_loc;
        if (vec16 && okr && c < k) {
          const double2 v = *reinterpret_cast<const double2*>(ws.W + g * k + c);
          w[i][j][0] = v.x; w[i][j][1] = v.y;
        } else {
          w[i][j][0] = (okr && c < k) ? ws.W[g * k + c] : 0.0;
          w[i][j][1] = (okr && c + 1 < k) ? ws.W[g * k + c + 1] : 0.0;
        }
      }
    }
    double acc[C::MI][C::NI][2];
#pragma unroll
    for (int i = 0; i < C::MI; ++i)
#pragma unroll
      for (int j = 0; j < C::NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    const double* xs = Xs + buf * C::XSTAGE;
#pragma unroll 4
    for (int kk = 0; kk < KP; kk += 4) {
      double a[C::MI], b[C::NI];
#pragma unroll
      for (int i = 0; i < C::MI; ++i) a[i] = xs[(wm * C::WM + i * 8 + (lane >> 2)) * C::LDX + kk + (lane & 3)];
#pragma unroll
      for (int j = 0; j < C::NI; ++j) b[j] = Cs[(kk + (lane & 3)) * C::LDC + wn * C::WN + j * 8 + (lane >> 2)];
#pragma unroll
      for (int i = 0; i < C::MI; ++i)
#pragma unroll
        for (int j = 0; j < C::NI; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
#pragma unroll
    for (int i = 0; i < C::MI; ++i) {
      const int64_t g = r0 + wm * C::WM + i * 8 + (lane >> 2);
      if (g >= ws.n_loc) continue;
#pragma unroll
      for (int j = 0; j < C::NI; ++j) {
        const int cl = wn * C::WN + j * 8 + 2 * (lane & 3), c = n0 + cl;
        const double x0 = __fma_rn(w[i][j][0], ssc[cl], -acc[i][j][0]);
        const double x1 = __fma_rn(w[i][j][1], ssc[cl + 1], -acc[i][j][1]);
        if (vec16 && c < k) {
          *reinterpret_cast<double2*>(out + g * k + c) = make_double2(x0, x1);
          if (NORM) {
            nacc[j][0] = __fma_rn(x0, x0, nacc[j][0]);
            nacc[j][1] = __fma_rn(x1, x1, nacc[j][1]);
          }
        } else {
          if (c < k) { out[g * k + c] = x0; if (NORM) nacc[j][0] = __fma_rn(x0, x0, nacc[j][0]); }
          if (c + 1 < k) { out[g * k + c + 1] = x1; if (NORM) nacc[j][1] = __fma_rn(x1, x1, nacc[j][1]); }
        }
      }
    }
  }
  if (!NORM) return;
  // column norm partials: slot rows (wm, lane/4) reduced in fixed order
#pragma unroll
  for (int j = 0; j < C::NI; ++j) {
    const int c = wn * C::WN + j * 8 + 2 * (lane & 3);
    sred[wm * 8 + (lane >> 2)][c] = nacc[j][0];
    sred[wm * 8 + (lane >> 2)][c + 1] = nacc[j][1];
  }
  __syncthreads();
  for (int j = tid; j < NC; j += C::THREADS) {
    double s = 0.0;
    for (int q = 0; q < WARPS_M * 8; ++q) s += sred[q][j];
    ws.nslot[(int64_t)blockIdx.x * KP + n0 + j] = s;
  }
}

// ---------------------------------------------------------------- pass C at k = 128, ping-pong
// A sweep's pass C (NORM = false) with two consumer groups of 8 warps that take alternate 32-row
// tiles: one group's epilogue (w s - acc, stores) overlaps the other group's DMMAs, instead of all
// 16 warps leaving the DMMA pipe idle together at every tile boundary.  The X tiles arrive as eight
// 128-byte-swizzled 16-column TMA boxes (the pass-B tensor map) in a 2-stage ring (stage = group);
// the last warp of a group through its tile's DMMAs refills the stage with the group's next tile (no
// producer warp: 16 warps keep 128 registers).  All of Csig stays resident (padded rows,
// conflict-free B fragments).  Same DMMA k-order and epilogue fma as passC_kernel (identical
// results); in place, rows >= top only.
// Generalised (round 2, late): ST ring stages shared by the two groups (tile j -> stage j % ST); with
// ST = 3 a group's next tile is issued by the OTHER group one tile earlier (PassCPP3: 24-row tiles).
template <int BR_, int ST_, int WM__, int WN__>
struct PassCPPCfgT {
  static constexpr int KP = 128, BR = BR_, GROUPS = 2, GWARPS = 8, ST = ST_;
  static constexpr int WARPS = GROUPS * GWARPS, THREADS = WARPS * 32, BLOCK = THREADS;
  static constexpr int WM_ = WM__, WN_ = WN__, WTM = BR / WM_, WTN = KP / WN_, MI = WTM / 8, NI = WTN / 8;
  static constexpr int LDC = KP + 8;
  static constexpr int BOX = BR * 128, STAGE = (KP / 16) * BOX;
  static constexpr int SMEM = ST * STAGE + KP * LDC * 8 + 1024 + 2 * ST * 8;
};
using PassCPPCfg = PassCPPCfgT<32, 2, 2, 4>;
using PassCPP3Cfg = PassCPPCfgT<24, 3, 1, 8>;
using PassCPP4Cfg = PassCPPCfgT<16, 4, 1, 8>;
template <class C>
__global__ void __launch_bounds__(C::BLOCK, 1)
passC_pp_kernel(Ws ws, const __grid_constant__ CUtensorMap tmX, double* __restrict__ out) {
  constexpr int BR = C::BR, KP = C::KP;
  extern __shared__ __align__(1024) unsigned char pcsm[];
  __shared__ double ssc[KP];
  griddep_wait();
  if (*ws.status != ST_OK) return;
  unsigned char* ring = smem_align1024(pcsm);
  double* Cs = reinterpret_cast<double*>(ring + C::ST * C::STAGE);
  uint64_t* full = reinterpret_cast<uint64_t*>(Cs + KP * C::LDC);
  int* done = reinterpret_cast<int*>(full + C::ST);                 // warps through a tile's DMMAs (monotonic)
  const int k = ws.k, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t rows = ws.n_loc - ws.top;
  const int64_t ntile = (rows + BR - 1) / BR;
  const int njt = (int)((ntile > blockIdx.x) ? (ntile - blockIdx.x + gridDim.x - 1) / gridDim.x : 0);   // this CTA's tiles
  auto issue = [&](int j) {   // tile j of this CTA -> stage j % ST
    const int s = j % C::ST;
    const int r0 = (int)(ws.top + (blockIdx.x + (int64_t)j * gridDim.x) * BR);
    mbar_expect_tx(&full[s], C::STAGE);
#pragma unroll
    for (int b = 0; b < KP / 16; ++b) tma_load_2d(ring + s * C::STAGE + b * C::BOX, &tmX, 16 * b, r0, &full[s]);
  };
  if (tid == 0) {
    for (int s = 0; s < C::ST; ++s) { mbar_init(&full[s], 1); done[s] = 0; }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    for (int j = 0; j < C::ST && j < njt; ++j) issue(j);
  }
  for (int e = tid; e < KP * KP; e += blockDim.x) {
    const int l = e / KP, j = e % KP;
    Cs[l * C::LDC + j] = (l < k && j < k) ? ws.Csig[l * k + j] : 0.0;
  }
  for (int j = tid; j < KP; j += blockDim.x) ssc[j] = (j < k) ? ws.scal[j] : 0.0;
  __syncthreads();
  const int grp = warp / C::GWARPS, gw = warp % C::GWARPS;
  const int wm = gw / C::WN_, wn = gw % C::WN_;
  for (int j = grp; j < njt; j += C::GROUPS) {
    const int s = j % C::ST;
    const int64_t r0 = ws.top + (blockIdx.x + (int64_t)j * gridDim.x) * BR;
    double w[C::MI][C::NI][2];   // this thread's W entries, loaded ahead of the MMAs
#pragma unroll
    for (int i = 0; i < C::MI; ++i) {
      const int64_t g = r0 + wm * C::WTM + i * 8 + (lane >> 2);
#pragma unroll
      for (int jn = 0; jn < C::NI; ++jn) {
        const int c = wn * C::WTN + jn * 8 + 2 * (lane & 3);
        if (g < ws.n_loc && c < k) {
          const double2 v = *reinterpret_cast<const double2*>(ws.W + g * k + c);
          w[i][jn][0] = v.x; w[i][jn][1] = v.y;
        } else {
          w[i][jn][0] = w[i][jn][1] = 0.0;
        }
      }
    }
    double acc[C::MI][C::NI][2];
#pragma unroll
    for (int i = 0; i < C::MI; ++i)
#pragma unroll
      for (int jn = 0; jn < C::NI; ++jn) acc[i][jn][0] = acc[i][jn][1] = 0.0;
    mbar_wait(&full[s], (j / C::ST) & 1);
    const unsigned char* xs = ring + s * C::STAGE;
#pragma unroll 4
    for (int kk = 0; kk < KP; kk += 4) {
      // the 4 k columns of this DMMA step: {2s, 2s + 1, 2s + 8, 2s + 9} of its 16-column box (s = (kk / 4) % 4),
      // two 16-byte chunks 4 apart, so the 8 rows x 4 columns of a fragment load hit distinct chunks under
      // the 128-byte swizzle (columns kk .. kk + 3 put rows r and r ^ 1 on the same chunks)
      const int t = lane & 3;
      const int kc = (kk & ~15) + 2 * ((kk >> 2) & 3) + (t & 1) + 8 * (t >> 1);
      double a[C::MI], b[C::NI];
#pragma unroll
      for (int i = 0; i < C::MI; ++i)
        a[i] = *reinterpret_cast<const double*>(xs + swz_off<BR>(wm * C::WTM + i * 8 + (lane >> 2), kc));
#pragma unroll
      for (int jn = 0; jn < C::NI; ++jn) b[jn] = Cs[kc * C::LDC + wn * C::WTN + jn * 8 + (lane >> 2)];
#pragma unroll
      for (int i = 0; i < C::MI; ++i)
#pragma unroll
        for (int jn = 0; jn < C::NI; ++jn) dmma(acc[i][jn][0], acc[i][jn][1], a[i], b[jn]);
    }
    __syncwarp();                                // this warp's reads of the stage are done
    if (lane == 0 && stage_release_last(&done[s], C::GWARPS) && j + C::ST < njt) issue(j + C::ST);   // last of the group
#pragma unroll
    for (int i = 0; i < C::MI; ++i) {
      const int64_t g = r0 + wm * C::WTM + i * 8 + (lane >> 2);
      if (g >= ws.n_loc) continue;
#pragma unroll
      for (int jn = 0; jn < C::NI; ++jn) {
        const int cl = wn * C::WTN + jn * 8 + 2 * (lane & 3);
        if (cl >= k) continue;
        const double x0 = __fma_rn(w[i][jn][0], ssc[cl], -acc[i][jn][0]);
        const double x1 = __fma_rn(w[i][jn][1], ssc[cl + 1], -acc[i][jn][1]);
        *reinterpret_cast<double2*>(out + g * k + cl) = make_double2(x0, x1);
      }
    }
  }
}

// x_ij *= 1/||x~_j||.  The thread count is a multiple of k/2 on the vector path, so every
// thread always scales the same column pair (no per-element index arithmetic).
__global__ void __launch_bounds__(256) normalize_kernel(Ws ws, double* __restrict__ X) {
  __shared__ double sinv[KMAX];
  __shared__ int sbad;
  griddep_wait();   // (programmatic dependent launch: the predecessor's writes are visible after this)
  if (*ws.status != ST_OK) return;
  const int k = ws.k;
  if (ws.multi) {         // combine the gathered per-rank column sums in rank order
    if (threadIdx.x == 0) sbad = 0;
    __syncthreads();
    for (int j = threadIdx.x; j < k; j += blockDim.x) {
      double sum = ws.nrm_all[j];
      for (int r = 1; r < ws.world; ++r) sum += ws.nrm_all[(int64_t)r * k + j];
      const double nrm = sqrt(sum);
      sinv[j] = 1.0 / nrm;
      if (!isfinite(sinv[j]) || !(nrm > 0.0)) sbad = 1;
      if (blockIdx.x == 0) ws.invn[j] = sinv[j];
    }
    __syncthreads();
    if (sbad) {
      if (blockIdx.x == 0 && threadIdx.x == 0) atomicCAS(ws.status, ST_OK, ST_DIVERGED);
      return;
    }
  }
  const double* invn = ws.multi ? sinv : ws.invn;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nthr = (int64_t)gridDim.x * blockDim.x;
  if ((k & 1) == 0 && (256 % (k / 2)) == 0 && ((uintptr_t)X & 15) == 0) {   // (X may be only 8-byte aligned)
    const int64_t total2 = ws.n_loc * (k / 2);
    const int j = (int)(tid % (k / 2)) * 2;
    const double s0 = invn[j], s1 = invn[j + 1];
    double2* X2 = reinterpret_cast<double2*>(X);
    const double2* T2 = reinterpret_cast<const double2*>(ws.Xt);
    for (int64_t e = tid; e < total2; e += nthr) {
      double2 v = T2[e];
      v.x *= s0; v.y *= s1;
      X2[e] = v;
    }
  } else {
    const int64_t total = ws.n_loc * k;
    for (int64_t e = tid; e < total; e += nthr) X[e] = ws.Xt[e] * invn[e % k];
  }
}

}  // namespace rf
