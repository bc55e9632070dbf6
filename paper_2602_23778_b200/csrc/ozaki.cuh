// ozaki.cuh -- S1 for dense A (W = A X^) with FP64 accuracy on the INT8 tensor cores
// (tcgen05.mma kind::i8), opt-in through refine_opts.emul.  Ozaki-style splitting:
//
//   A_ij = 2^{e_i + 2} sum_{t=1..S} a^(t)_ij 2^{-8t} + r_ij,   X_lj = 2^{f_j + 2} sum_{u=1..S} x^(u)_lj 2^{-8u} + q_lj
//
// with int8 slices a^(t), x^(u) the BALANCED base-256 digits (in [-128, 127]; the leading one in
// [-64, 64]) of the 64-bit integer N = rint(v 2^{8S-2-e}) (|N| <= 2^{8S-2}; one exact FP64 scaling,
// one F2I, then integer byte extraction with carry), e_i the exponent of row i's max |A_ij| (A is
// constant: sliced once at init, 2^{-e_i} |.| < 1) and f_j that of column j's max |X_lj| (every
// sweep).  Then
//
//   (A X)_ij = 2^{e_i + f_j + 4} sum_{c=2..S+1} 2^{-8c} L_c[i][j],   L_c = sum_{t+u=c} a^(t) x^(u)
//
// where every L_c is an exact integer product accumulated in int32 on the tensor cores (|L_c| <=
// (c-1) 128^2 K, K <= OZ_KMAX keeps it below 2^31) and combined in FP64.  Dropped terms (t + u >
// S + 1) and the roundings are below ~7 2^{4-8S} (S = 7: 2^-52) of max|A_i.| max|X_.j| per product
// term.  Unlike FP64 rounding this error is relative to the row / column MAXIMA, so entries
// far below their row's largest lose relative accuracy (the classic limit of the scheme).  The
// diagonal -- the dominant entry of the diagonally dominant and near-diagonal (Q ~ I) matrices the
// method meets -- is therefore taken out: it is not sliced (e_i is the OFF-diagonal row maximum)
// and a_ii x_ij is added in FP64 in the epilogue.  Rows whose off-diagonal entries span a wider
// dynamic range than the sweep tolerates need the DMMA path (emul = 0, the default).  Balanced
// 8-bit digits carry 8 bits per int8 (7 for sign-magnitude digits): 7 slices give the 54 bits that
// 8 sign-magnitude slices gave, with 28 slice products instead of 36 and 7/8 of the bytes.
//
// Per K step of 32 the MMA for slice t of A multiplies the concatenated X slices u = 1 .. S+1-t
// (N = m k <= 256) into the TMEM accumulators of levels t+1 .. t+m, which are laid out contiguously
// by level -- so the S(S+1)/2 slice products take 2S-ish MMAs.  Tiles are pre-arranged in HBM in the
// UMMA canonical K-major layout (8-row x 16-byte core matrices): A as [row tile][K step][slice]
// [128 x 32] (one contiguous 4S KB bulk copy per K step), X as [K step][slice][k x 32].
#pragma once
#include "common.cuh"
#include "tc_passes.cuh"

namespace rf {

constexpr int OZ_S = 7;                     // slices per operand (balanced base-256 digits)
constexpr int OZ_BM = 128, OZ_BK = 32;      // A rows per tile, K per MMA (int8)
constexpr int OZ_KMAX = 16384;              // K per CTA: 7 * 128^2 * 16384 < 2^31 (exact int32 levels)
constexpr uint32_t OZ_SBO = (OZ_BK / 16) * 128;            // 8-row groups: 256 B
constexpr uint32_t OZ_ATILE = OZ_BM * OZ_BK;               // 4 KB per A slice tile
constexpr int OZ_STAGES = 4;
constexpr int OZ_THREADS = 256;             // warp 0: producer, warp 1: MMA issue, warps 4-7: epilogue

RF_DEV constexpr uint32_t oz_off(int r, int kk) {   // element (row r, K kk) of a canonical int8 tile
  return (uint32_t)(r / 8) * OZ_SBO + (uint32_t)(kk / 16) * 128u + (uint32_t)(r % 8) * 16u + (uint32_t)(kk % 16);
}
RF_DEV int oz_exponent(double m) {          // smallest e with m < 2^e (m >= 0); 0 for m == 0
  if (!(m > 0.0)) return 0;
  int e;
  frexp(m, &e);                             // m = f 2^e, f in [0.5, 1)
  return e;
}
// balanced base-256 digits of v 2^{-e} (|v| < 2^e): N = rint(v 2^{8S-2-e}), |N| <= 2^{8S-2}, split
// from the least significant byte up -- d_t = the signed low byte of N (in [-128, 127]), N <- (N - d_t)
// / 256 (exact) -- so N = sum_t d_t 2^{8(S-t)} and the leading digit |d_1| <= 64 (+ 0.502) fits.
RF_DEV void oz_slices_e(double v, int e, int8_t (&d)[OZ_S]) {
  int64_t N = __double2ll_rn(ldexp(v, 8 * OZ_S - 2 - e));   // exact scaling, rounded to nearest
#pragma unroll
  for (int t = OZ_S - 1; t >= 1; --t) {
    const int8_t lo = (int8_t)(uint8_t)(N & 255);
    d[t] = lo;
    N = (N - lo) >> 8;
  }
  d[0] = (int8_t)N;
}

// ---- init: per-row exponent of A (row max) -------------------------------------------------
// (off-diagonal max; local row i is global row row0 + i) and the diagonal entries in FP64
__global__ void __launch_bounds__(256) oz_rowexp_kernel(const double* __restrict__ A, int64_t lda, int64_t M,
                                                        int64_t n, int64_t row0, int32_t* __restrict__ e,
                                                        double* __restrict__ diag) {
  const int lane = threadIdx.x & 31;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < M;
       i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    double m = 0.0;
    for (int64_t j = lane; j < n; j += 32)
      if (j != row0 + i) m = fmax(m, fabs(A[i * lda + j]));
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) {
      e[i] = oz_exponent(m);
      diag[i] = (row0 + i < n) ? A[i * lda + row0 + i] : 0.0;
    }
  }
}

// ---- init: A slices, tiles [rt][ks][t][128 x 32] (zero padded past M rows / n columns) ---------
// one thread per (row, 16-column chunk): 16 FP64 -> S uint4 stores
__global__ void __launch_bounds__(256) oz_slice_A_kernel(const double* __restrict__ A, int64_t lda, int64_t M,
                                                         int64_t n, int64_t row0, const int32_t* __restrict__ e,
                                                         int8_t* __restrict__ As, int64_t nks) {
  const int64_t nrt = (M + OZ_BM - 1) / OZ_BM;
  const int64_t nchunk = nks * (OZ_BK / 16);           // 16-column chunks per row
  const int64_t total = nrt * OZ_BM * nchunk;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < total; g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = g / nchunk, ch = g % nchunk;     // row, chunk (consecutive threads: same row)
    const int64_t ks = ch / (OZ_BK / 16);
    const int kk0 = (int)(ch % (OZ_BK / 16)) * 16;
    uint32_t w[OZ_S][4];
#pragma unroll
    for (int t = 0; t < OZ_S; ++t) w[t][0] = w[t][1] = w[t][2] = w[t][3] = 0u;
    if (i < M) {
      const int ei = e[i];
#pragma unroll 4
      for (int q = 0; q < 16; ++q) {
        const int64_t j = ks * OZ_BK + kk0 + q;
        int8_t d[OZ_S];
        oz_slices_e((j < n && j != row0 + i) ? A[i * lda + j] : 0.0, ei, d);   // diagonal: FP64 epilogue
#pragma unroll
        for (int t = 0; t < OZ_S; ++t) w[t][q >> 2] |= (uint32_t)(uint8_t)d[t] << (8 * (q & 3));
      }
    }
    const int64_t rt = i / OZ_BM;
    int8_t* tile0 = As + ((rt * nks + ks) * OZ_S) * (int64_t)OZ_ATILE;
    const uint32_t off = oz_off((int)(i % OZ_BM), kk0);
#pragma unroll
    for (int t = 0; t < OZ_S; ++t)
      *reinterpret_cast<uint4*>(tile0 + t * OZ_ATILE + off) = make_uint4(w[t][0], w[t][1], w[t][2], w[t][3]);
  }
}

// ---- per sweep: column exponents of X (n x k), atomicMax of exact exponents (order-free) -------
__global__ void __launch_bounds__(256) oz_colexp_kernel(const double* __restrict__ X, int64_t n, int k,
                                                        int32_t* __restrict__ f) {
  // f[] preset to INT_MIN by the caller (memset 0x80)
  const int j = threadIdx.x % k, rows_per = blockDim.x / k;
  double m = 0.0;
  for (int64_t l = (int64_t)blockIdx.x * rows_per + threadIdx.x / k; l < n; l += (int64_t)gridDim.x * rows_per)
    m = fmax(m, fabs(X[l * k + j]));
  if ((int)threadIdx.x < rows_per * k) atomicMax(&f[j], oz_exponent(m));
}

// ---- per sweep: X slices, tiles [ks][u][k x 32]: element (n = j, K = l) -----------------------
__global__ void __launch_bounds__(256) oz_slice_X_kernel(const double* __restrict__ X, int64_t n, int k,
                                                         const int32_t* __restrict__ f, int8_t* __restrict__ Xs,
                                                         int64_t nks) {
  const int64_t total = nks * OZ_BK * (int64_t)k;      // one thread per (K row l, column j)
  const int64_t tile = (int64_t)k * OZ_BK;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < total; g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t l = g / k;
    const int j = (int)(g % k);
    int8_t d[OZ_S];
    oz_slices_e(l < n ? X[l * k + j] : 0.0, f[j], d);
    const int64_t ks = l / OZ_BK;
    const uint32_t off = oz_off(j, (int)(l % OZ_BK));
#pragma unroll
    for (int u = 0; u < OZ_S; ++u) Xs[(ks * OZ_S + u) * tile + off] = d[u];
  }
}

// ---- the GEMM: out[blockIdx.y][m][j] = partial (A X)_mj over K steps [ks0, ks1) ---------------
// grid (row tiles, splits); one CTA per SM.  K-chunk per split <= OZ_KMAX.
template <int KK>   // k (multiple of 16, <= 64)
struct OzCfg {
  static constexpr uint32_t XTILE = KK * OZ_BK;                            // bytes per X slice tile
  static constexpr uint32_t STAGE = OZ_S * OZ_ATILE + OZ_S * XTILE;       // A slices + X slices
  static constexpr int SMEM = 1024 + OZ_STAGES * STAGE;
  static constexpr int MAXM = 256 / KK;                                   // X slices per MMA (N <= 256)
  static constexpr int TCOLS = OZ_S * KK <= 256 ? 256 : 512;              // TMEM columns (levels x k)
};

template <int KK>
__global__ void __launch_bounds__(OZ_THREADS, 1) oz_gemm_kernel(const int8_t* __restrict__ As,
                                                                const int8_t* __restrict__ Xs,
                                                                const int32_t* __restrict__ e,
                                                                const int32_t* __restrict__ f, int64_t M,
                                                                int64_t nks, int64_t ks_per, double* __restrict__ out,
                                                                int64_t out_split_stride, const double* __restrict__ diag,
                                                                const double* __restrict__ Xd, int64_t row0,
                                                                const int* __restrict__ status) {
  using C = OzCfg<KK>;
  extern __shared__ __align__(16) unsigned char oz_raw[];
  __shared__ __align__(8) uint64_t full[OZ_STAGES], empty[OZ_STAGES], accb;
  __shared__ uint32_t tmem_base;
  griddep_wait();   // (programmatic dependent launch: the predecessor's writes are visible after this)
  if (*status != ST_OK) return;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t rt = blockIdx.x;
  const int64_t ks0 = (int64_t)blockIdx.y * ks_per;
  const int64_t ks1 = (ks0 + ks_per < nks) ? ks0 + ks_per : nks;
  const int nst = (ks1 > ks0) ? (int)(ks1 - ks0) : 0;
  unsigned char* base = oz_raw + ((1024 - (smem_u32(oz_raw) & 1023)) & 1023);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base)),
                 "r"(C::TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    for (int i = 0; i < OZ_STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(&accb, 1);
  }
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base;
  if (warp == 0) {                                   // ---- producer: one stage = A slices + X slices
    if (lane == 0) {
      for (int t = 0; t < nst; ++t) {
        const int s = t % OZ_STAGES;
        if (t >= OZ_STAGES) mbar_wait(&empty[s], ((t / OZ_STAGES) - 1) & 1);
        const int64_t ks = ks0 + t;
        unsigned char* st = base + s * C::STAGE;
        mbar_expect_tx(&full[s], C::STAGE);
        bulk_g2s(st, As + ((rt * nks + ks) * OZ_S) * (int64_t)OZ_ATILE, OZ_S * OZ_ATILE, &full[s]);
        bulk_g2s(st + OZ_S * OZ_ATILE, Xs + ks * OZ_S * (int64_t)C::XTILE, OZ_S * C::XTILE, &full[s]);
      }
    }
  } else if (warp == 1) {                            // ---- MMA issue (one thread)
    if (lane == 0) {
      for (int t = 0; t < nst; ++t) {
        const int s = t % OZ_STAGES;
        mbar_wait(&full[s], (t / OZ_STAGES) & 1);
        tc_fence_after();
        const uint32_t sa = smem_u32(base + s * C::STAGE), sx = sa + OZ_S * OZ_ATILE;
#pragma unroll
        for (int ta = 1; ta <= OZ_S; ++ta) {         // slice t of A x slices u = 1 .. S + 1 - t of X
          const uint64_t da = umma_desc(sa + (ta - 1) * OZ_ATILE, 128, OZ_SBO);
          for (int u0 = 1; u0 <= OZ_S + 1 - ta; u0 += C::MAXM) {
            const int m = (OZ_S + 1 - ta - u0 + 1) < C::MAXM ? (OZ_S + 1 - ta - u0 + 1) : C::MAXM;
            const uint64_t db = umma_desc(sx + (u0 - 1) * C::XTILE, 128, OZ_SBO);
            const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)((m * KK) >> 3) << 17) |
                                   ((uint32_t)(OZ_BM >> 4) << 24);
            const uint32_t dcol = tmem + (uint32_t)((ta + u0 - 2) * KK);   // level c = ta + u0 at column (c - 2) k
            const uint32_t acc = (t > 0 || ta > 1) ? 1u : 0u;            // ta = 1 initialises every level
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(dcol),
                "l"(da), "l"(db), "r"(idesc), "r"(acc));
          }
        }
        umma_commit(&empty[s]);                       // the stage's smem may be refilled
      }
      umma_commit(&accb);
    }
  } else if (warp >= 4) {                            // ---- epilogue: TMEM lane (row) 32 (w - 4) + lane
    const int r = 32 * (warp - 4) + lane;
    const int64_t i = rt * OZ_BM + r;
    if (nst > 0) mbar_wait(&accb, 0);
    tc_fence_after();
    const uint32_t tl = tmem + ((uint32_t)(32 * (warp - 4)) << 16);
    const double se = (i < M) ? ldexp(1.0, e[i]) : 0.0;
    double* o = out + (int64_t)blockIdx.y * out_split_stride + i * KK;
#pragma unroll 1
    for (int c0 = 0; c0 < KK; c0 += 16) {
      double acc[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) acc[q] = 0.0;
      if (nst > 0) {
#pragma unroll 1
        for (int c = OZ_S + 1; c >= 2; --c) {          // smallest levels first
          float v[16];
          tmem_ld16(tl + (uint32_t)((c - 2) * KK + c0), v);
          const double w = ldexp(1.0, 4 - 8 * c);
#pragma unroll
          for (int q = 0; q < 16; ++q) acc[q] = fma((double)(int32_t)__float_as_uint(v[q]), w, acc[q]);
        }
      }
      if (i < M) {   // split 0 adds the FP64 diagonal term a_ii x_ij
        const double di = blockIdx.y == 0 ? diag[i] : 0.0;
        const double* xr = Xd + (row0 + i) * KK + c0;
#pragma unroll
        for (int q = 0; q < 16; q += 2) {
          const double2 xv = *reinterpret_cast<const double2*>(xr + q);
          *reinterpret_cast<double2*>(o + c0 + q) =
              make_double2(fma(di, xv.x, acc[q] * se * ldexp(1.0, f[c0 + q])),
                           fma(di, xv.y, acc[q + 1] * se * ldexp(1.0, f[c0 + q + 1])));
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(C::TCOLS));
}

}  // namespace rf

namespace rf {

// ---- pass C on the INT8 tensor cores (k = 128; refine_opts.emul) ------------------------------
// x~_i = w_i s - x_i Csig for rows i >= top.  x_i Csig is the sweep's O(residual) correction, so it
// needs ~1e-8 relative accuracy for the 1e-10 one-step parity (4 digits measured 1.03e-10 on the
// 3-D Laplacian with a 1.8e-5 gap) and none beyond that for the final FP64 accuracy (it vanishes at
// convergence): SC = 5 slices of 7 bits per operand (~2^-35 of the maxima), levels c <= 6.
// Transposed product per 32-row slab:
//   D[j][i] = sum_l Csig[l][j] x_il = 2^{g_j + h_i} sum_{c=2..5} 2^{-7c} L_c[j][i]
// with g_j the exponent of column j of Csig (A = Csig^T sliced once per CTA) and h_i that of row i
// of X (found by the converter from the slab: no global pass), L_c exact int32 sums (K = 128).
// The MMA for slice t of A takes the concatenated X slices u = 1 .. SC+1-t (N = 32 (SC+1-t)) and
// writes levels t+1 .. SC+1, laid out by level in TMEM (2 buffers x 5 levels x 32 columns).
constexpr int OZC_S = 5, OZC_TN = 32, OZC_NS = 3, OZC_K = 128;
constexpr int OZC_CONV = 128, OZC_EPI = 128, OZC_THREADS = OZC_CONV + OZC_EPI + 32 + 32;   // + producer, MMA
constexpr uint32_t OZC_SBO = (OZC_K / 16) * 128;                 // 1024 B: 8-row groups of a K = 128 tile
constexpr uint32_t OZC_ATILE = 128 * OZC_K;                      // 16 KB per slice of Csig^T
constexpr uint32_t OZC_BTILE = OZC_TN * OZC_K;                   // 4 KB per slice of a slab
constexpr uint32_t OZC_BBUF = OZC_S * OZC_BTILE;                 // 16 KB
constexpr uint32_t OZC_SLOT = OZC_TN * OZC_K * 8;                // 32 KB of X rows
constexpr int OZC_TCOLS = 512;                                   // 2 x 5 levels x 32 columns (power of 2)
constexpr int OZC_SMEM = 1024 + OZC_S * OZC_ATILE + 2 * OZC_BBUF + OZC_NS * OZC_SLOT;   // 217 KB
RF_DEV constexpr uint32_t ozc_off(int r, int l) {               // element (row r, K l), K = 128 int8 tile
  return (uint32_t)(r / 8) * OZC_SBO + (uint32_t)(l / 16) * 128u + (uint32_t)(r % 8) * 16u + (uint32_t)(l % 16);
}
RF_DEV void ozc_digits(double v, int e, int8_t (&d)[OZC_S]) {   // |v| 2^-e truncated to 7 SC bits, base 128
  const uint64_t M = (uint64_t)(fabs(v) * ldexp(1.0, 7 * OZC_S - e));
  const bool neg = v < 0.0;
#pragma unroll
  for (int t = 0; t < OZC_S; ++t) {
    const int q = (int)((M >> (7 * (OZC_S - 1 - t))) & 127u);
    d[t] = (int8_t)(neg ? -q : q);
  }
}

__global__ void __launch_bounds__(OZC_THREADS, 1) passC_oz_kernel(Ws ws, const double* X, double* out) {
  extern __shared__ __align__(16) unsigned char ozc_raw[];
  __shared__ __align__(8) uint64_t full[OZC_NS], empty[OZC_NS], opfree[2], cvd[2], accf[2], acce[2];
  __shared__ uint32_t tmem_base;
  __shared__ double ssc[OZC_K];
  __shared__ int32_t sg[OZC_K];                 // column exponents of Csig
  __shared__ int32_t sh[4][OZC_TN];             // row exponents of slab t in sh[t % 4] (read by its
                                                // epilogue before it releases TMEM; slab t + 4's
                                                // converter runs only after that, via opfree / acce)
  griddep_wait();   // (programmatic dependent launch: the predecessor's writes are visible after this)
  if (*ws.status != ST_OK) return;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int k = ws.k;                           // == 128
  const int64_t rows = ws.n_loc - ws.top;
  const int64_t per = ((rows + gridDim.x - 1) / gridDim.x + OZC_TN - 1) / OZC_TN * OZC_TN;
  const int64_t rb = ws.top + (int64_t)blockIdx.x * per;
  const int64_t re = (rb + per < ws.n_loc) ? rb + per : ws.n_loc;
  const int nst = (re > rb) ? (int)((re - rb + OZC_TN - 1) / OZC_TN) : 0;
  unsigned char* base = ozc_raw + ((1024 - (smem_u32(ozc_raw) & 1023)) & 1023);
  unsigned char* As = base;                                           // [SC][128 j x 128 l]
  unsigned char* Bs = base + OZC_S * OZC_ATILE;                       // [2][SC][32 rows x 128 l]
  unsigned char* F = Bs + 2 * OZC_BBUF;                               // [NS][32 X rows] FP64
  if (tid < OZC_K) {                            // A = Csig^T, row j scaled by 2^-g_j
    double m = 0.0;
    for (int l = 0; l < k; ++l) m = fmax(m, fabs(ws.Csig[l * k + tid]));
    sg[tid] = oz_exponent(m);
    ssc[tid] = ws.scal[tid];
  }
  __syncthreads();
  for (int e = tid; e < OZC_K * OZC_K / 4; e += OZC_THREADS) {     // 4 consecutive l per thread
    const int j = e % OZC_K, l0 = 4 * (e / OZC_K);
    uint32_t w[OZC_S];
#pragma unroll
    for (int t = 0; t < OZC_S; ++t) w[t] = 0u;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      int8_t d[OZC_S];
      ozc_digits(ws.Csig[(l0 + q) * k + j], sg[j], d);
#pragma unroll
      for (int t = 0; t < OZC_S; ++t) w[t] |= (uint32_t)(uint8_t)d[t] << (8 * q);
    }
#pragma unroll
    for (int t = 0; t < OZC_S; ++t) *reinterpret_cast<uint32_t*>(As + t * OZC_ATILE + ozc_off(j, l0)) = w[t];
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base)),
                 "r"(OZC_TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    for (int i = 0; i < OZC_NS; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], OZC_CONV / 32);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&opfree[i], 1);
      mbar_init(&cvd[i], OZC_CONV);
      mbar_init(&accf[i], 1);
      mbar_init(&acce[i], OZC_EPI / 32);
    }
  }
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base;
  double nacc = 0.0;
  if (warp == (OZC_CONV + OZC_EPI) / 32) {         // ---- producer: X rows of each slab
    if (lane == 0) {
      for (int t = 0; t < nst; ++t) {
        const int s = t % OZC_NS;
        if (t >= OZC_NS) {
          mbar_wait(&empty[s], ((t / OZC_NS) - 1) & 1);
          fence_async_smem();                       // converters' generic reads of slot s -> the refill
        }
        const int64_t r0 = rb + (int64_t)t * OZC_TN;
        const uint32_t bytes = (uint32_t)min((int64_t)OZC_TN, re - r0) * OZC_K * 8;
        mbar_expect_tx(&full[s], bytes);
        bulk_g2s(F + s * OZC_SLOT, X + r0 * OZC_K, bytes, &full[s]);
      }
    }
  } else if (warp < OZC_CONV / 32) {               // ---- converters (warp w: slab rows 8w .. 8w+7) + MMA
    for (int t = 0; t < nst; ++t) {
      const int s = t % OZC_NS, o = t & 1;
      mbar_wait(&full[s], (t / OZC_NS) & 1);
      if (t >= 2) mbar_wait(&opfree[o], ((t >> 1) - 1) & 1);          // B buffer o read by slab t-2's MMAs
      const int nr = (int)min((int64_t)OZC_TN, re - (rb + (int64_t)t * OZC_TN));
      const double* fx = reinterpret_cast<const double*>(F + s * OZC_SLOT);
      unsigned char* B = Bs + o * OZC_BBUF;
      // warp w owns slab rows 8w .. 8w+7.  (1) row exponents: lanes read 4 values of a row each,
      // redux.max of the exponents; (2) digits: lane (r8 = lane / 4, c = lane % 4) converts values
      // 16 g + 4 c .. +3 of row 8w + r8, so one store instruction fills a whole 8-row x 16-byte core
      // matrix (32 distinct banks)
      constexpr int RPW = OZC_TN / 4;               // rows per converter warp (8)
#pragma unroll 2
      for (int rr = 0; rr < RPW; ++rr) {
        const int r = RPW * warp + rr;
        double m = 0.0;
        if (r < nr) {
          const double2 a0 = reinterpret_cast<const double2*>(fx + r * OZC_K)[2 * lane];
          const double2 a1 = reinterpret_cast<const double2*>(fx + r * OZC_K)[2 * lane + 1];
          m = fmax(fmax(fabs(a0.x), fabs(a0.y)), fmax(fabs(a1.x), fabs(a1.y)));
        }
        const int h = __reduce_max_sync(0xffffffffu, oz_exponent(m) + 2048) - 2048;   // row exponent
        if (lane == 0) sh[t & 3][r] = h;
      }
      __syncwarp();
      {
        const int r = RPW * warp + (lane >> 2), c = lane & 3;
        const int h = sh[t & 3][r];
        const bool ok = r < nr;
#pragma unroll 2
        for (int g = 0; g < OZC_K / 16; ++g) {
          const int l0 = 16 * g + 4 * c;
          double2 a0 = make_double2(0.0, 0.0), a1 = make_double2(0.0, 0.0);
          if (ok) {
            a0 = *reinterpret_cast<const double2*>(fx + r * OZC_K + l0);
            a1 = *reinterpret_cast<const double2*>(fx + r * OZC_K + l0 + 2);
          }
          const double v[4] = {a0.x, a0.y, a1.x, a1.y};
          uint32_t w[OZC_S];
#pragma unroll
          for (int u = 0; u < OZC_S; ++u) w[u] = 0u;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            int8_t d[OZC_S];
            ozc_digits(v[q], h, d);
#pragma unroll
            for (int u = 0; u < OZC_S; ++u) w[u] |= (uint32_t)(uint8_t)d[u] << (8 * q);
          }
#pragma unroll
          for (int u = 0; u < OZC_S; ++u) *reinterpret_cast<uint32_t*>(B + u * OZC_BTILE + ozc_off(r, l0)) = w[u];
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);      // the slab's X rows are consumed
      fence_async_smem();                         // digit stores -> the tensor core's async proxy
      mbar_arrive(&cvd[o]);
    }
  } else if (warp == (OZC_CONV + OZC_EPI) / 32 + 1) {   // ---- MMA issue (one thread), decoupled from the converters
    if (lane == 0) {
      const uint32_t sa = smem_u32(As);
      for (int t = 0; t < nst; ++t) {
        const int o = t & 1;
        mbar_wait(&cvd[o], (t >> 1) & 1);                              // B buffer o converted
        if (t >= 2) mbar_wait(&acce[o], ((t >> 1) - 1) & 1);          // TMEM buffer o read out
        tc_fence_after();
        const uint32_t sb = smem_u32(Bs + o * OZC_BBUF);
        const uint32_t td = tmem + (uint32_t)(o * OZC_S * OZC_TN);
#pragma unroll
        for (int kk = 0; kk < OZC_K / 32; ++kk) {
#pragma unroll
          for (int ta = 1; ta <= OZC_S; ++ta) {   // A slice t x X slices 1 .. SC+1-t -> levels t+1 .. SC+1
            const int m = OZC_S + 1 - ta;
            const uint64_t da = umma_desc(sa + (ta - 1) * OZC_ATILE + kk * 256, 128, OZC_SBO);
            const uint64_t db = umma_desc(sb + kk * 256, 128, OZC_SBO);
            const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)((m * OZC_TN) >> 3) << 17) |
                                   ((uint32_t)(128 >> 4) << 24);
            const uint32_t acc = (kk > 0 || ta > 1) ? 1u : 0u;
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(td + (uint32_t)((ta - 1) * OZC_TN)),
                "l"(da), "l"(db), "r"(idesc), "r"(acc));
          }
        }
        umma_commit(&opfree[o]);
        umma_commit(&accf[o]);
      }
    }
  } else {                                         // ---- epilogue: column j = 32 (warp % 4) + lane
    const int j = 32 * (warp & 3) + lane;
    const double sj = ssc[j];
    const int gj = sg[j];
    const uint32_t tl = tmem + ((uint32_t)(32 * (warp & 3)) << 16);
    for (int t = 0; t < nst; ++t) {
      const int o = t & 1;
      const int64_t r0 = rb + (int64_t)t * OZC_TN;
      const int nr = (int)min((int64_t)OZC_TN, re - r0);
      mbar_wait(&accf[o], (t >> 1) & 1);
      tc_fence_after();
#pragma unroll 1
      for (int h0 = 0; h0 < OZC_TN; h0 += 16) {    // 16 rows at a time (registers)
        double w[16], acc[16];
#pragma unroll
        for (int r = 0; r < 16; ++r) {
          w[r] = (h0 + r < nr) ? __ldcs(ws.W + (r0 + h0 + r) * OZC_K + j) : 0.0;
          acc[r] = 0.0;
        }
#pragma unroll
        for (int c = OZC_S + 1; c >= 2; --c) {       // smallest levels first
          float v[16];
          tmem_ld16(tl + (uint32_t)(o * OZC_S * OZC_TN + (c - 2) * OZC_TN + h0), v);
          const double wc = ldexp(1.0, -7 * c);
#pragma unroll
          for (int r = 0; r < 16; ++r) acc[r] = fma((double)(int32_t)__float_as_uint(v[r]), wc, acc[r]);
        }
#pragma unroll
        for (int r = 0; r < 16; ++r) {
          if (h0 + r < nr) {
            const double p2 = __longlong_as_double((long long)(1023 + gj + sh[t & 3][h0 + r]) << 52);   // 2^(g + h)
            const double x = __fma_rn(w[r], sj, -(acc[r] * p2));
            __stcs(out + (r0 + h0 + r) * OZC_K + j, x);
            nacc = __fma_rn(x, x, nacc);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acce[o]);
    }
  }
  __syncthreads();
  if (warp >= OZC_CONV / 32 && warp < (OZC_CONV + OZC_EPI) / 32)
    ws.nslot[(int64_t)blockIdx.x * OZC_K + (tid - OZC_CONV)] = nacc;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(OZC_TCOLS));
}

}  // namespace rf
