// kxk.cuh -- the serial k x k stages of a sweep, each one CTA of 1024 threads (k <= 128).
//
// kxk_rq + kxk_lu (S2 + S3): fixed-order reduction of the alpha/g double-double partials
//            -> alpha_j, d_j = g_j / alpha_j (eq. Rayleigh, Alg. 4
//            lines 3-4); modified LU of the top k x k block X^_1 in shared memory (Alg. 2,
//            PAPER.md:271-284, sign(0) = +1) -> Sigma, U, Y_1 = L;  U^{-1} and L^{-1} by
//            blocked triangular inversion;  T = -U Sigma Y_1^{-T} = -(U Sigma) (L^{-1})^T
//            (Alg. 3).  Rows l > k of Alg. 2 only read U's rows, so
//            Y_2 = X^_2 U^{-1} (the tall-skinny triangular apply) is never formed on the
//            hot path: it is applied through k x k algebra.
// kxk_finish (S4-S6 top block + all k x k algebra): with the one-time flip
//            X' = X^ Sigma, W' = W Sigma, U' = U Sigma (reading R2),
//            U'^{-1} = Sigma U^{-1}:
//              R_1  = W'_1 - X'_1 D                              (line 5 operand)
//              Z    = Y^T R = L^T R_1 + U'^{-T} M'               M' = X'_2^T R_2 (pass B)
//              P    = T^T Z,   V_1 = R_1 - L P                   (V = H^T R)
//              E_11 = (1-alpha)/2 | beta | V_1/(d_j - d_i)       (line 6)
//              P~   = U'^{-1} P
//              Y_2^T E_2 = U'^{-T} (M' - G' P~) D^{-1}          G' = X'_2^T X'_2 (pass B)
//              Qm   = Y^T E = L^T E_11 + Y_2^T E_2,  B = T Qm   (line 7)
//              X~_1 = X'_1 + (E_11 - L B)                        (top rows, written here)
//              C'   = P~ D^{-1} + U'^{-1} B,  Csig = Sigma C'    (pass C: x~_i = w_i Sigma D^{-1} - x_i Csig)
//            plus the sweep statistics.
// All k x k products go through cta_gemm: operands live in global scratch (L2-resident),
// 32-deep K panels are staged in shared memory and multiplied with DMMA m8n8k4 (one warp
// per 8 x 8 output tile).  Triangular inverses use 16 x 16 diagonal blocks solved in registers and
// recursive doubling with cta_gemm.
#pragma once
#include "common.cuh"

namespace rf {

constexpr int KXK_THREADS = 1024;
__device__ long long* g_gemm_tlog = nullptr;   // optional phase log of one cta_gemm call (timing builds)
__device__ long long* g_fullk_tlog = nullptr;  // ... and of the first two cta_gemm_fullk calls
__device__ long long* g_fullk_tlog_first = nullptr;
constexpr int PANEL = 32;
constexpr int LDA_P = PANEL + 4;                  // As[i][p]: A-fragment reads (8 rows x 4) conflict-free
constexpr int LDB_P = KMAX + 8;                   // Bs[p][j]: B-fragment reads (4 rows x 8) conflict-free
constexpr int PANEL_SMEM = KMAX * LDA_P + PANEL * LDB_P;   // doubles of shared memory cta_gemm needs

// C (M x N, ldc) = alpha op(A) op(B) + beta C0 on the FP64 tensor cores (DMMA m8n8k4).
// op(A) is M x K, op(B) is K x N, M, N <= 128.  K is consumed in 32-deep panels staged in
// shared memory; warp w owns the 8 x 8 output tiles w, w + 32, ...  C0 may alias C (each
// element is read then written by the same thread).  Starts and ends with a barrier.
template <int MAXT>
__device__ __noinline__ void cta_gemm_t(int M, int N, int K, double alpha, const double* A, int lda, bool ta,
                                        const double* B, int ldb, bool tb, double beta, const double* C0, int ldc0,
                                        double* C, int ldc, double* sm) {
  double* As = sm;                      // [KMAX][LDA_P]  As[i][p] = op(A)(i, kk+p)
  double* Bs = sm + KMAX * LDA_P;       // [PANEL][LDB_P] Bs[p][j] = op(B)(kk+p, j)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tm = (M + 7) >> 3, tn = (N + 7) >> 3, ntile = tm * tn;
  double acc[MAXT][2];
#pragma unroll
  for (int t = 0; t < MAXT; ++t) acc[t][0] = acc[t][1] = 0.0;
  const int Mp = tm * 8, Np = tn * 8;
  const bool glob = __isGlobal(A) && __isGlobal(B);
  const bool blk = (MAXT == 8) && tm == 16 && tn == 16;
  const int bi0 = (warp >> 2) * 16, bj0 = (warp & 3) * 32;
  long long* tl = g_gemm_tlog;
  int ts = 0;
  if (tl && tid == 0) tl[ts] = clock64();
  ++ts;
  for (int kk = 0; kk < K; kk += PANEL) {
    const int pk = min(PANEL, K - kk);
    __syncthreads();
    if (tl && tid == 0 && ts < 14) tl[ts] = clock64();
    ++ts;
    // stage op(A)(0:Mp, kk:kk+32) and op(B)(kk:kk+32, 0:Np), zero-padded.  Global operands go
    // through cp.async (every copy of the panel in flight at once: one L2 round trip per panel,
    // not one per element); shared-memory operands (kxk_lu's small-k factors) are copied directly.
    if (glob) {
      for (int e = tid; e < PANEL * Mp; e += KXK_THREADS) {
        int i, p;
        if (ta) { i = e % Mp; p = e / Mp; } else { p = e & (PANEL - 1); i = e >> 5; }
        const bool ok = p < pk && i < M;
        cp_async8(As + i * LDA_P + p, ok ? (ta ? A + (kk + p) * lda + i : A + i * lda + kk + p) : A, ok);
      }
      for (int e = tid; e < PANEL * Np; e += KXK_THREADS) {
        int j, p;
        if (tb) { p = e & (PANEL - 1); j = e >> 5; } else { j = e % Np; p = e / Np; }
        const bool ok = p < pk && j < N;
        cp_async8(Bs + p * LDB_P + j, ok ? (tb ? B + j * ldb + kk + p : B + (kk + p) * ldb + j) : B, ok);
      }
      cp_async_commit();
      cp_async_wait<0>();
    } else {
      for (int e = tid; e < PANEL * Mp; e += KXK_THREADS) {
        int i, p;
        if (ta) { i = e % Mp; p = e / Mp; } else { p = e & (PANEL - 1); i = e >> 5; }
        As[i * LDA_P + p] = (p < pk && i < M) ? (ta ? A[(kk + p) * lda + i] : A[i * lda + kk + p]) : 0.0;
      }
      for (int e = tid; e < PANEL * Np; e += KXK_THREADS) {
        int j, p;
        if (tb) { p = e & (PANEL - 1); j = e >> 5; } else { j = e % Np; p = e / Np; }
        Bs[p * LDB_P + j] = (p < pk && j < N) ? (tb ? B[j * ldb + kk + p] : B[(kk + p) * ldb + j]) : 0.0;
      }
    }
    __syncthreads();
    if (tl && tid == 0 && ts < 14) tl[ts] = clock64();
    ++ts;
    if (blk) {   // 16 x 16 tiles: warp w owns a 2 x 4 block (A / B fragments reused 4 / 2 times)
#pragma unroll
      for (int p = 0; p < PANEL; p += 4) {
        double a[2], b[4];
#pragma unroll
        for (int r = 0; r < 2; ++r) a[r] = As[(bi0 + 8 * r + (lane >> 2)) * LDA_P + p + (lane & 3)];
#pragma unroll
        for (int c = 0; c < 4; ++c) b[c] = Bs[(p + (lane & 3)) * LDB_P + bj0 + 8 * c + (lane >> 2)];
#pragma unroll
        for (int t = 0; t < (MAXT == 8 ? 8 : 0); ++t) dmma(acc[t][0], acc[t][1], a[t >> 2], b[t & 3]);
      }
    } else {
#pragma unroll
      for (int t = 0; t < MAXT; ++t) {
        const int tile = warp + 32 * t;
        if (tile < ntile) {
          const int i0 = (tile / tn) * 8, j0 = (tile % tn) * 8;
#pragma unroll
          for (int p = 0; p < PANEL; p += 4) {
            const double a = As[(i0 + (lane >> 2)) * LDA_P + p + (lane & 3)];
            const double b = Bs[(p + (lane & 3)) * LDB_P + j0 + (lane >> 2)];
            dmma(acc[t][0], acc[t][1], a, b);
          }
        }
      }
    }
  }
#pragma unroll
  for (int t = 0; t < MAXT; ++t) {
    const int tile = warp + 32 * t;
    if (blk || tile < ntile) {
      const int i = blk ? bi0 + 8 * (t >> 2) + (lane >> 2) : (tile / tn) * 8 + (lane >> 2);
      const int j = blk ? bj0 + 8 * (t & 3) + 2 * (lane & 3) : (tile % tn) * 8 + 2 * (lane & 3);
#pragma unroll
      for (int h = 0; h < 2; ++h)
        if (i < M && j + h < N) {
          const double v = alpha * acc[t][h];
          C[i * ldc + j + h] = (beta != 0.0) ? fma(beta, C0[i * ldc0 + j + h], v) : v;
        }
    }
  }
  if (tl && tid == 0 && ts < 14) tl[ts] = clock64();
  __syncthreads();
  if (tl && tid == 0 && ts < 15) { tl[ts + 1] = clock64(); tl[15] = ts + 2; }
  if (tl && tid == 0) g_gemm_tlog = nullptr;       // log only the first call
}

// tiles per warp: 1 (<= 32 output tiles, k <= 44), 2 (k <= 64), 8 (k <= 128).  Instantiating
// by tile count keeps the unrolled MMA body small, so it stays in the instruction cache of the
// single SM that runs the k x k chain.
__device__ __forceinline__ void cta_gemm(int M, int N, int K, double alpha, const double* A, int lda, bool ta,
                                         const double* B, int ldb, bool tb, double beta, const double* C0, int ldc0,
                                         double* C, int ldc, double* sm) {
  const int nt = ((M + 7) >> 3) * ((N + 7) >> 3);
  if (nt <= 32) cta_gemm_t<1>(M, N, K, alpha, A, lda, ta, B, ldb, tb, beta, C0, ldc0, C, ldc, sm);
  else if (nt <= 64) cta_gemm_t<2>(M, N, K, alpha, A, lda, ta, B, ldb, tb, beta, C0, ldc0, C, ldc, sm);
  else cta_gemm_t<8>(M, N, K, alpha, A, lda, ta, B, ldb, tb, beta, C0, ldc0, C, ldc, sm);
}

// Row block of a k x k product for kxk_finish's cluster CTAs: C (M x N) = alpha op(A) B + beta C0
// with M <= 32, N, K <= 128, op(A) and B staged WHOLE (all K) in shared memory by one burst of
// cp.async copies (one L2 round trip per product instead of one per 32-deep panel).  Warp w owns
// output tiles w and w + 32.  Starts and ends with a barrier.
constexpr int FK_SMEM = 32 * (KMAX + 4) + KMAX * (KMAX + 8);   // doubles
// bulk-copy staging of cta_gemm_fullk: an mbarrier and its phase, set up by kxk_finish_body (g_fk_bulk)
__shared__ uint64_t g_fk_mbar;
__shared__ uint32_t g_fk_phase;
__shared__ int g_fk_bulk;
// Dual form (A2 != nullptr): also C2 = alpha2 op(A2) B + beta2 C02 with the same B, staged once; the
// 2 ntile output tiles are dealt over the warps (so a k = 128 row block of 8 rows keeps all 32 warps busy).
__device__ __noinline__ void cta_gemm_fullk(int M, int N, int K, double alpha, const double* A, int lda, bool ta,
                                            const double* B, int ldb, double beta, const double* C0, int ldc0,
                                            double* C, int ldc, double* sm, const double* A2 = nullptr,
                                            double alpha2 = 0.0, double beta2 = 0.0, const double* C02 = nullptr,
                                            double* C2 = nullptr) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tm = (M + 7) >> 3, tn = (N + 7) >> 3, ntile = tm * tn;
  const int nA = A2 ? 2 : 1;
  const int Mp = tm * 8, Np = tn * 8, Kp = (K + 3) & ~3;
  const int lda_s = Kp + 4, ldb_s = Np + 8;
  double* As = sm;                      // [nA][Mp][lda_s]  As[a][i][p] = op(A_a)(i, p)
  double* Bs = sm + nA * Mp * lda_s;    // [Kp][ldb_s]      Bs[p][j] = B(p, j)
  long long* fl = g_fullk_tlog;
  if (fl && tid == 0) fl[0] = clock64();
  const uint32_t par = g_fk_phase & 1;   // (before the barrier: thread 0 advances the phase after it)
  __syncthreads();
  const bool v16 = ((K | N | M | lda | ldb) & 1) == 0 && (((uintptr_t)A | (uintptr_t)B | (uintptr_t)(A2 ? A2 : A)) & 15) == 0;
  const bool glob = __isGlobal(A) && __isGlobal(B) && (!A2 || __isGlobal(A2));
  auto zero_pad = [&]() {   // K, M, N are multiples of 8 on the clustered path except a ragged k: pad explicitly
    for (int a = 0; a < nA; ++a) {
      double* Aa = As + a * Mp * lda_s;
      #pragma unroll 1
      for (int e = tid; e < Mp * (Kp - K) + (Mp - M) * Kp; e += KXK_THREADS) {
        if (e < Mp * (Kp - K)) Aa[(e / (Kp - K)) * lda_s + K + e % (Kp - K)] = 0.0;
        else { const int f = e - Mp * (Kp - K); Aa[(M + f / Kp) * lda_s + f % Kp] = 0.0; }
      }
    }
    #pragma unroll 1
    for (int e = tid; e < (Kp - K) * Np + K * (Np - N); e += KXK_THREADS) {
      if (e < (Kp - K) * Np) Bs[(K + e / Np) * ldb_s + e % Np] = 0.0;
      else { const int f = e - (Kp - K) * Np; Bs[(f / (Np - N)) * ldb_s + N + f % (Np - N)] = 0.0; }
    }
  };
  auto stage_At = [&](const double* Aa, double* dst) {   // op(A)(i, p) = A[p][i]: element-wise transpose
    #pragma unroll 1
    for (int e = tid; e < M * K; e += KXK_THREADS) {
      const int p = e / M, i = e - p * M;
      cp_async8(dst + i * lda_s + p, Aa + (size_t)p * lda + i, true);
    }
  };
  if (g_fk_bulk && glob && v16) {
    // one 1-D bulk copy (cp.async.bulk, the TMA engine) per row of B and of A (A not transposed), all
    // completing on one mbarrier: ~160 row copies instead of ~9,000 16-byte cp.async per product
    // (measured 3.4 - 6 us of staging per k = 128 product with cp.async)
    if (tid == 0) mbar_expect_tx(&g_fk_mbar, (uint32_t)(K * N * 8 + (ta ? 0 : nA * M * K * 8)));
    if (tid < K || (!ta && tid < K + nA * M)) {
      asm volatile("fence.proxy.async;\n" ::: "memory");   // generic writes (this cluster's, acquired) -> async reads
      if (tid < K) {
        bulk_g2s(Bs + tid * ldb_s, B + (size_t)tid * ldb, (uint32_t)(N * 8), &g_fk_mbar);
      } else {
        const int a = (tid - K) / M, i = (tid - K) - a * M;
        bulk_g2s(As + (a * Mp + i) * lda_s, (a ? A2 : A) + (size_t)i * lda, (uint32_t)(K * 8), &g_fk_mbar);
      }
    }
    if (ta) {
      stage_At(A, As);
      if (A2) stage_At(A2, As + Mp * lda_s);
    }
    zero_pad();
    cp_async_commit();
    cp_async_wait<0>();
    mbar_wait(&g_fk_mbar, par);
    if (tid == 0) ++g_fk_phase;   // (every thread read it before the entry barrier)
  } else if (glob && v16) {
    // 16-byte copies, (row, column-pair) walked without divisions (one per thread up front): the
    // 8-byte / division form cost ~10 us per k = 128 product, mostly issue
    {   // B: K rows x N / 2 pairs
      const int n2 = N / 2, step = KXK_THREADS;
      int p = tid / n2, j = tid - p * n2;
      const int dp = step / n2, dj = step - dp * n2;
      for (int e = tid; e < K * n2; e += step) {
        cp_async16(Bs + p * ldb_s + 2 * j, B + (size_t)p * ldb + 2 * j, true);
        p += dp; j += dj;
        if (j >= n2) { j -= n2; ++p; }
      }
    }
    for (int a = 0; a < nA; ++a) {
      const double* Aa = a ? A2 : A;
      double* dst = As + a * Mp * lda_s;
      if (!ta) {   // op(A) = A: M rows x K / 2 pairs
        const int k2 = K / 2;
        int i = tid / k2, q = tid - i * k2;
        const int di = KXK_THREADS / k2, dq = KXK_THREADS - di * k2;
        for (int e = tid; e < M * k2; e += KXK_THREADS) {
          cp_async16(dst + i * lda_s + 2 * q, Aa + (size_t)i * lda + 2 * q, true);
          i += di; q += dq;
          if (q >= k2) { q -= k2; ++i; }
        }
      } else {
        stage_At(Aa, dst);
      }
    }
    zero_pad();
    cp_async_commit();
    cp_async_wait<0>();
  } else {
    for (int a = 0; a < nA; ++a) {
      const double* Aa = a ? A2 : A;
      double* dst = As + a * Mp * lda_s;
      for (int e = tid; e < Mp * Kp; e += KXK_THREADS) {
        int i, p;
        if (ta) { i = e % Mp; p = e / Mp; } else { p = e % Kp; i = e / Kp; }
        dst[i * lda_s + p] = (p < K && i < M) ? (ta ? Aa[p * lda + i] : Aa[i * lda + p]) : 0.0;
      }
    }
    for (int e = tid; e < Kp * Np; e += KXK_THREADS) {
      const int j = e % Np, p = e / Np;
      Bs[p * ldb_s + j] = (p < K && j < N) ? B[p * ldb + j] : 0.0;
    }
  }
  __syncthreads();
  if (fl && tid == 0) fl[1] = clock64();
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    const int tt = warp + 32 * t;
    if (tt < nA * ntile) {
      const int a = tt >= ntile ? 1 : 0, tile = tt - a * ntile;
      const int i0 = (tile / tn) * 8, j0 = (tile % tn) * 8;
      double c0 = 0.0, c1 = 0.0;
      const double* ap = As + (a * Mp + i0 + (lane >> 2)) * lda_s + (lane & 3);
      const double* bp = Bs + (lane & 3) * ldb_s + j0 + (lane >> 2);
#pragma unroll 8
      for (int p = 0; p < Kp; p += 4) dmma(c0, c1, ap[p], bp[p * ldb_s]);
      const int i = i0 + (lane >> 2), j = j0 + 2 * (lane & 3);
      const double al = a ? alpha2 : alpha, be = a ? beta2 : beta;
      const double* Ci = a ? C02 : C0;
      double* Co = a ? C2 : C;
      if (i < M) {
        if (j < N) Co[i * ldc + j] = (be != 0.0) ? fma(be, Ci[i * ldc0 + j], al * c0) : al * c0;
        if (j + 1 < N) Co[i * ldc + j + 1] = (be != 0.0) ? fma(be, Ci[i * ldc0 + j + 1], al * c1) : al * c1;
      }
    }
  }
  if (fl && tid == 0) fl[2] = clock64();
  __syncthreads();
  if (fl && tid == 0) { fl[3] = clock64(); g_fullk_tlog = (fl == g_fullk_tlog_first) ? fl + 4 : nullptr; }   // log the first two calls
}

// Inverse of a k x k triangular matrix S (ld k) into R (ld k).  upper: S upper triangular;
// else unit lower (diagonal taken as 1).  tmp: k x k scratch.  16 x 16 diagonal blocks are
// inverted by substitution in registers (one thread per column), then off-diagonal blocks are
// filled level by level: upper  R12 = -R11 S12 R22;  lower  R21 = -R22 S21 R11.
__device__ void cta_trinv(int k, const double* S, bool upper, double* R, double* tmp, double* sm) {
  constexpr int BS = 16;
  const int tid = threadIdx.x;
  for (int e = tid; e < k * k; e += KXK_THREADS) R[e] = 0.0;
  __syncthreads();
  if (tid < k) {
    const int c = tid, b0 = (c / BS) * BS, bn = min(BS, k - b0), cl = c - b0;
    double x[BS];
#pragma unroll
    for (int i = 0; i < BS; ++i) x[i] = 0.0;
    if (upper) {
#pragma unroll
      for (int i = BS - 1; i >= 0; --i) {
        if (i < bn && i <= cl) {
          double s = (i == cl) ? 1.0 : 0.0;
#pragma unroll
          for (int l = i + 1; l < BS; ++l)
            if (l < bn && l <= cl) s = fma(-S[(b0 + i) * k + b0 + l], x[l], s);
          x[i] = s / S[(b0 + i) * k + b0 + i];
        }
      }
    } else {
#pragma unroll
      for (int i = 0; i < BS; ++i) {
        if (i < bn && i >= cl) {
          double s = (i == cl) ? 1.0 : 0.0;
#pragma unroll
          for (int l = 0; l < BS; ++l)
            if (l < i && l >= cl) s = fma(-S[(b0 + i) * k + b0 + l], x[l], s);
          x[i] = s;
        }
      }
    }
#pragma unroll
    for (int i = 0; i < BS; ++i)
      if (i < bn) R[(b0 + i) * k + c] = x[i];
  }
  __syncthreads();
  for (int s = BS; s < k; s *= 2) {
    for (int b0 = 0; b0 + s < k; b0 += 2 * s) {
      const int b1 = b0 + s, n1 = s, n2 = min(s, k - b1);
      if (upper) {   // R12 = -R11 (S12 R22)
        cta_gemm(n1, n2, n2, 1.0, S + b0 * k + b1, k, false, R + b1 * k + b1, k, false, 0.0, nullptr, 0,
                 tmp, k, sm);
        cta_gemm(n1, n2, n1, -1.0, R + b0 * k + b0, k, false, tmp, k, false, 0.0, nullptr, 0, R + b0 * k + b1, k,
                 sm);
      } else {       // R21 = -R22 (S21 R11)
        cta_gemm(n2, n1, n1, 1.0, S + b1 * k + b0, k, false, R + b0 * k + b0, k, false, 0.0, nullptr, 0,
                 tmp, k, sm);
        cta_gemm(n2, n1, n2, -1.0, R + b1 * k + b1, k, false, tmp, k, false, 0.0, nullptr, 0, R + b1 * k + b0, k,
                 sm);
      }
    }
  }
}

// alpha/g slot reduction: P parts per column (contiguous slot ranges, 4 interleaved accumulators
// each), then a fixed pairwise tree over the parts.  On return pa[j], pg[j] (j < k) hold the
// column sums.  Called by the whole block.
__device__ void reduce_ag_slots(const Ws& ws, dd* pa, dd* pg) {
  const int k = ws.k, tid = threadIdx.x, nt = KXK_THREADS;
  const int P = nt / k;
  const int j = tid % k, p = tid / k;
  dd a = {0.0, 0.0}, g = {0.0, 0.0};
  if (p < P) {
    const int s0 = (int)((int64_t)ws.n_ag * p / P), s1 = (int)((int64_t)ws.n_ag * (p + 1) / P);
    dd a4[4] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}}, g4[4] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
    int s = s0;
    for (; s + 8 <= s1; s += 8) {
      double v[8][4];
#pragma unroll
      for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int q = 0; q < 4; ++q) v[u][q] = ws.ag[((int64_t)(s + u) * k + j) * 4 + q];
#pragma unroll
      for (int u = 0; u < 8; ++u) { dd_add(a4[u & 3], dd{v[u][0], v[u][1]}); dd_add(g4[u & 3], dd{v[u][2], v[u][3]}); }
    }
    for (; s < s1; ++s) {
      const double* slot = ws.ag + ((int64_t)s * k + j) * 4;
      dd_add(a4[0], dd{slot[0], slot[1]});
      dd_add(g4[0], dd{slot[2], slot[3]});
    }
    a = a4[0]; g = g4[0];
#pragma unroll
    for (int u = 1; u < 4; ++u) { dd_add(a, a4[u]); dd_add(g, g4[u]); }
  }
  pa[tid] = a;
  pg[tid] = g;
  __syncthreads();
  for (int st = 1; st < P; st *= 2) {
    if (p < P && (p % (2 * st)) == 0 && p + st < P) {
      dd_add(pa[tid], pa[tid + st * k]);
      dd_add(pg[tid], pg[tid + st * k]);
    }
    __syncthreads();
  }
}

// world > 1: this rank's alpha/g double-double vector (4 doubles per column) for the all-gather
__global__ void __launch_bounds__(KXK_THREADS) ag_local_kernel(Ws ws) {
  __shared__ dd pa[KXK_THREADS], pg[KXK_THREADS];
  griddep_wait();   // (programmatic dependent launch: the predecessor's writes are visible after this)
  if (*ws.status != ST_OK) return;
  reduce_ag_slots(ws, pa, pg);
  if (threadIdx.x < ws.k) {
    double* v = ws.ag_send + 4 * threadIdx.x;
    v[0] = pa[threadIdx.x].hi; v[1] = pa[threadIdx.x].lo; v[2] = pg[threadIdx.x].hi; v[3] = pg[threadIdx.x].lo;
  }
}

// ---------------------------------------------------------------- kxk_rq (S2: alpha, Rayleigh quotients)
// body shared by kxk_rq_kernel and sweep_tail_kernel (tail_small.cuh): pa, pg: KXK_THREADS dd each
__device__ void kxk_rq_body(const Ws& ws, dd* pa, dd* pg, int& s_bad) {
  RF_TSTAMP(ws, 0);
  const int k = ws.k, tid = threadIdx.x, nt = KXK_THREADS;

  // 1. alpha_j, g_j: this rank's slots, or (world > 1) the gathered per-rank
  //    double-double vectors combined in rank order -- identical on every rank
  if (tid == 0) s_bad = ST_OK;
  if (ws.multi) {
    if (tid < k) {
      dd ta = {ws.ag_all[4 * tid], ws.ag_all[4 * tid + 1]}, tg = {ws.ag_all[4 * tid + 2], ws.ag_all[4 * tid + 3]};
      for (int r = 1; r < ws.world; ++r) {
        const double* v = ws.ag_all + (int64_t)r * 4 * k + 4 * tid;
        dd_add(ta, dd{v[0], v[1]});
        dd_add(tg, dd{v[2], v[3]});
      }
      pa[tid] = ta;
      pg[tid] = tg;
    }
    __syncthreads();
  } else {
    reduce_ag_slots(ws, pa, pg);
  }
  if (tid < k) {
    const double al = dd_val(pa[tid]), gv = dd_val(pg[tid]);
    const double dj = gv / al;
    ws.alpha[tid] = al;
    ws.d[tid] = dj;
    ws.rd[tid] = 1.0 / dj;
    int bad = ST_OK;
    if (!isfinite(al) || !isfinite(dj)) bad = ST_DIVERGED;
    else if (!(al > 0.0)) bad = ST_E_INVALID;
    else if (fabs(dj) <= ws.delta) bad = ST_E_NEAR_ZERO_RQ;
    if (bad != ST_OK) atomicCAS(&s_bad, ST_OK, bad);
  }
  RF_TSTAMP(ws, 1);
  __syncthreads();
  if (tid == 0 && s_bad != ST_OK) atomicCAS(ws.status, ST_OK, s_bad);
}
__global__ void __launch_bounds__(KXK_THREADS) kxk_rq_kernel(Ws ws) {
  __shared__ dd pa[KXK_THREADS], pg[KXK_THREADS];
  __shared__ int s_bad;
  griddep_wait();   // (programmatic dependent launch: the predecessor's writes are visible after this)
  if (*ws.status != ST_OK) return;
  kxk_rq_body(ws, pa, pg, s_bad);
}

// ---------------------------------------------------------------- kxk_lu
// S3 on the top k x k block: needs only X^_1, so it runs on a side stream concurrently with
// S1 / S2 / passB (joined before kxk_finish).  Rank 0 only.
// Shared memory: Q (k x k, the in-place modified LU); for k <= 64 also Ls, Ts, Us (L, T, U^{-1}).
// body shared by kxk_lu_kernel and sweep_tail_kernel; Q: max(4 k^2 (k <= 64) or k^2, PANEL_SMEM) doubles
__device__ void kxk_lu_body(const Ws& ws, const double* __restrict__ Xtop, double* Q, int& s_bad) {
  const int k = ws.k, tid = threadIdx.x, nt = KXK_THREADS;
  for (int e = tid; e < k * k; e += nt) Q[e] = Xtop[e];
  if (tid == 0) s_bad = ST_OK;

  // 2. Alg. 2 on the top block, literal arithmetic: sigma_j = -sign(q_jj) (sign(0)=+1),
  //    q_jj -= sigma_j, q_lj /= q_jj, q_lh -= q_lj q_jh.  One barrier per step: thread (l, h)
  //    forms q_lj / pivot itself, column j of Y goes straight to L (never re-read here), and
  //    only q_lh with l, h > j are written, which no other thread reads during the step.
  const bool small = (k <= 64);
  double* Ls = Q + k * k;          // small k: L, T, U^{-1} also in shared memory
  double* Ts = Q + 2 * k * k;
  double* Us = Q + 3 * k * k;
  __syncthreads();
  for (int jj = 0; jj < k; ++jj) {
    const double q = Q[jj * k + jj];
    const double s = (q >= 0.0) ? -1.0 : 1.0;
    const double piv = __dadd_rn(q, -s);
    if (piv == 0.0) {                       // uniform across the block
      if (tid == 0) atomicCAS(&s_bad, ST_OK, ST_E_ZERO_PIVOT);
      break;
    }
    if (tid == 0) ws.sigma[jj] = s;
    for (int l = jj + 1 + (tid >> 5); l < k; l += 32) {
      const double ql = __ddiv_rn(Q[l * k + jj], piv);
      for (int h = jj + (tid & 31); h < k; h += 32) {
        if (h == jj) {
          ws.L[l * k + jj] = ql;
          if (small) Ls[l * k + jj] = ql;
        } else {
          Q[l * k + h] = __dadd_rn(Q[l * k + h], -__dmul_rn(ql, Q[jj * k + h]));
        }
      }
    }
    __syncthreads();
  }
  __syncthreads();
  if (s_bad == ST_E_ZERO_PIVOT) {
    if (tid == 0) atomicCAS(ws.status, ST_OK, s_bad);
    return;
  }
  // U = upper(Q) with the shifted diagonal; L unit lower (strict part written above)
  for (int r = tid >> 5; r < k; r += 32)
    for (int c = tid & 31; c < k; c += 32) {
      const double qv = Q[r * k + c];
      const double sg = ws.sigma[r];
      const double u = (c > r) ? qv : (c == r ? __dadd_rn(qv, -sg) : 0.0);
      Q[r * k + c] = u;                                    // Q now holds U
      ws.U[r * k + c] = u;
      if (c >= r) {
        ws.L[r * k + c] = (c == r) ? 1.0 : 0.0;
        if (small) Ls[r * k + c] = (c == r) ? 1.0 : 0.0;
      }
    }
  __syncthreads();
  RF_TSTAMP(ws, 2);
  if (small) {
    // 3a. T = -U Sigma L^{-T}: thread i < k owns row i (t_ic = -u_ic s_c - sum_{i<=l<c} t_il L_cl);
    //     thread k + c owns column c of U^{-1} (back substitution).  All operands in shared memory.
    if (tid < k) {
      const int i = tid;
      for (int c = 0; c < i; ++c) Ts[i * k + c] = 0.0;
      for (int c = i; c < k; ++c) {
        double t = -(Q[i * k + c] * ws.sigma[c]);
        for (int l = i; l < c; ++l) t = fma(-Ts[i * k + l], Ls[c * k + l], t);
        Ts[i * k + c] = t;
      }
    } else if (tid < 2 * k) {
      const int c = tid - k;
      for (int i = k - 1; i > c; --i) Us[i * k + c] = 0.0;
      for (int i = c; i >= 0; --i) {
        double x = (i == c) ? 1.0 : 0.0;
        for (int l = i + 1; l <= c; ++l) x = fma(-Q[i * k + l], Us[l * k + c], x);
        Us[i * k + c] = x / Q[i * k + i];
      }
    }
    __syncthreads();
    for (int e = tid; e < k * k; e += nt) { ws.T[e] = Ts[e]; ws.Uinv[e] = Us[e]; }
  } else {
    // 3b. large k: blocked triangular inversion and a DMMA product through L2-resident scratch
    double* Up = ws.scratch;                   // U Sigma
    for (int r = tid >> 5; r < k; r += 32)
      for (int c = tid & 31; c < k; c += 32) Up[r * k + c] = Q[r * k + c] * ws.sigma[c];
    double* Linv = ws.scratch + k * k;
    double* tmp = ws.scratch + 2 * k * k;
    __syncthreads();
    cta_trinv(k, ws.U, true, ws.Uinv, tmp, Q);
    cta_trinv(k, ws.L, false, Linv, tmp, Q);
    cta_gemm(k, k, k, -1.0, Up, k, false, Linv, k, true, 0.0, nullptr, 0, ws.T, k, Q);
  }
  if (ws.kxk_h) {
    // the T products of kxk_finish's chain, moved off its critical path (this kernel overlaps S1 /
    // S2 / pass B on the side stream).  With U'^{-1} = Sigma U^{-1}:
    //   P = T^T (L^T R_1 + U'^{-T} M')  =>  V_1 = R_1 - H1^T R_1 - H3^T M',  P~ = H2^T R_1 + H4^T M'
    //   B = T (L^T E_11 + U'^{-T} S2)   =>  L B = H1 E_11 + H2 S2,          U'^{-1} B = H3 E_11 + H4 S2
    // with H1 = L T L^T, H2 = L T U'^{-T}, H3 = U'^{-1} T L^T, H4 = U'^{-1} T U'^{-T} (identities exact in
    // real arithmetic; every factor O(1) for near-orthonormal X^, so no cancellation is introduced).
    const int kk = k * k;
    double* H = ws.scratch + 16 * kk;
    double *LT = ws.scratch + 20 * kk, *UT = ws.scratch + 21 * kk, *UiS = ws.scratch + 22 * kk;
    __syncthreads();
    for (int e = tid; e < kk; e += nt) UiS[e] = ws.sigma[e / k] * ws.Uinv[e];
    cta_gemm(k, k, k, 1.0, ws.L, k, false, ws.T, k, false, 0.0, nullptr, 0, LT, k, Q);       // L T
    cta_gemm(k, k, k, 1.0, UiS, k, false, ws.T, k, false, 0.0, nullptr, 0, UT, k, Q);        // U'^{-1} T
    cta_gemm(k, k, k, 1.0, LT, k, false, ws.L, k, true, 0.0, nullptr, 0, H, k, Q);           // H1
    cta_gemm(k, k, k, 1.0, LT, k, false, UiS, k, true, 0.0, nullptr, 0, H + kk, k, Q);       // H2
    cta_gemm(k, k, k, 1.0, UT, k, false, ws.L, k, true, 0.0, nullptr, 0, H + 2 * kk, k, Q);  // H3
    cta_gemm(k, k, k, 1.0, UT, k, false, UiS, k, true, 0.0, nullptr, 0, H + 3 * kk, k, Q);   // H4
  }
  RF_TSTAMP(ws, 5);
  if (tid == 0 && s_bad != ST_OK) atomicCAS(ws.status, ST_OK, s_bad);
}
__global__ void __launch_bounds__(KXK_THREADS) kxk_lu_kernel(Ws ws, const double* __restrict__ Xtop) {
  extern __shared__ __align__(16) double Q[];
  __shared__ int s_bad;
  griddep_wait();   // (programmatic dependent launch: the predecessor's writes are visible after this)
  if (*ws.status != ST_OK) return;
  kxk_lu_body(ws, Xtop, Q, s_bad);
}

// ---------------------------------------------------------------- kxk_finish
// One thread-block cluster of kxk_cluster(k) CTAs (1024 threads each): CTA r owns rows
// [r0, r1) of every k x k result (a multiple of 8 rows), so each cta_gemm call computes its row
// block (M = r1 - r0) and the elementwise steps run on its rows; barrier.cluster (release /
// acquire: global-memory results of the other CTAs become visible) separates dependent phases.
// The per-column statistics and norms run on CTA 0.  k <= 32 runs as a single CTA.
RF_DEV unsigned cluster_ctarank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
RF_DEV unsigned cluster_nctarank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;\n" : "=r"(r));
  return r;
}
__device__ __noinline__ void cluster_sync() {   // (noinline: one copy in the instruction cache)
  if (cluster_nctarank() == 1) {   // single CTA: a block barrier orders its global accesses too
    __syncthreads();
    return;
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
// CTAs of kxk_finish's cluster: 16 (a non-portable cluster size) for k > 64, where the products are DMMA-
// throughput bound on 8 SMs (k = 128: 4.7 us per product of 16 x 128 x 128 per CTA); rows per CTA stay a
// multiple of 8, so k <= 64 gains nothing from more than 8
__host__ __device__ constexpr int kxk_cluster(int k, bool allow16 = true) {
  return k > 64 ? (allow16 ? 16 : 8) : (k >= 64 ? 8 : (k >= 32 ? 4 : 1));
}
constexpr int KXK_SCRATCH_MATS = 26;    // k x k scratch matrices: kxk_finish 0..15, H1..H4 16..19, kxk_lu temps 20..22, column partials 24..25
constexpr int KXK_SCRATCH_EXTRA = 64;   // doubles after them (cluster partials)

// Small k (k <= KXK_SMALL): the whole k x k chain in ONE CTA with every k x k operand resident in
// shared memory and each product one output element per thread (a plain fma chain over ascending p):
// no cluster barriers, no global scratch round trips and no per-product panel staging -- the chain is
// latency bound at these sizes (measured 29 us at k = 4, 39 us at k = 16 with the DMMA / L2-scratch form).
constexpr int KXK_SMALL = 32;
constexpr int KXK_SMALL_MATS = 20;   // k x k matrices resident in shared memory (see kxk_finish_kernel<true>)
// layout: 20 k x k matrices | column-sum partials (8 x 7 x k) | d copy (k) | sigma, d, alpha, rr2 (4 k) | 64 spare
__host__ __device__ constexpr int kxk_small_smem_doubles(int k) { return KXK_SMALL_MATS * k * k + 8 * 7 * k + k + 4 * k + 64; }
__device__ __noinline__ void smem_mm(int k, double alpha, const double* A, bool ta, const double* B, double beta, const double* C0,
                    double* C) {
  __syncthreads();
  const int t = threadIdx.x;
  if (t < k * k) {
    const int i = t / k, j = t - i * k;
    const double* a = ta ? A + i : A + i * k;
    const int as = ta ? k : 1;
    double acc = 0.0;
#pragma unroll 4
    for (int p = 0; p < k; ++p) acc = fma(a[p * as], B[p * k + j], acc);
    const double v = alpha * acc;
    C[i * k + j] = (beta != 0.0) ? fma(beta, C0[i * k + j], v) : v;
  }
  __syncthreads();
}

// Xtop/Wtop: the top k rows of X^ (in/out) and W (un-flipped), ld k.
// SMALL (k <= KXK_SMALL, one CTA): scratch, L, T, E_11 and X~_1 live in shared memory, products by smem_mm.
template <bool SMALL>
__device__ void kxk_finish_body(const Ws& ws, double* __restrict__ Xtop, const double* __restrict__ Wtop, double* sm,
                                int& s_hits, double (*s_red)[KMAX]) {
  const int k = ws.k, kk = k * k, tid = threadIdx.x, nt = KXK_THREADS;
  const int crank = SMALL ? 0 : (int)cluster_ctarank(), ncl = SMALL ? 1 : (int)cluster_nctarank();
  const int per = (((k + ncl - 1) / ncl) + 7) & ~7;
  const int r0 = min(k, crank * per), r1 = min(k, r0 + per), nr = r1 - r0;
  double* S = SMALL ? sm : ws.scratch;
  double *Xp = S, *R1 = S + kk, *Mp = S + 2 * kk, *Gp = S + 3 * kk, *Ui = S + 4 * kk, *Z = S + 5 * kk,
         *P = S + 6 * kk, *V1 = S + 7 * kk, *Pt = S + 8 * kk, *GPt = S + 9 * kk, *S2 = S + 10 * kk,
         *Qm = S + 11 * kk, *B = S + 12 * kk, *LB = S + 13 * kk, *UB = S + 14 * kk;
  // SMALL: copies of L, T and the CTA's E_11 / X~_1 in shared memory (matrices 15..17)
  const double* Lm = SMALL ? S + 16 * kk : ws.L;
  const double* Tm = SMALL ? S + 17 * kk : ws.T;
  double* E11 = SMALL ? S + 18 * kk : ws.E11;
  double* Xt1 = SMALL ? S + 19 * kk : ws.Xt;
  double* part = SMALL ? sm + kxk_small_smem_doubles(k) - 64 : S + KXK_SCRATCH_MATS * kk;   // [0, 16): delta hits, [16, 32): gram max
  const bool useH = !SMALL && ws.kxk_h;                // the precomputed H1..H4 of kxk_lu (scratch + 16 k^2)
  const double* H = S + 16 * kk;
  double* cs_base = SMALL ? S + KXK_SMALL_MATS * kk : sm;   // column-sum partials (after the matrices when SMALL)
  double* vec = cs_base + 8 * 7 * k + k;               // SMALL: sigma, d, alpha, rr2 copies
  const double* sig = SMALL ? vec : ws.sigma;
  const double* d = SMALL ? vec + k : ws.d;
  const double* alp = SMALL ? vec + 2 * k : ws.alpha;
  const double* rr2p = SMALL ? vec + 3 * k : ws.rr2;
  // this CTA's rows of C = alpha op(A) B + beta C0 (k x k operands, B not transposed)
  auto rgemm = [&](double alpha, const double* A, bool ta, const double* Bm, double beta, const double* C0, double* C) {
    if (SMALL) {
      smem_mm(k, alpha, A, ta, Bm, beta, C0, C);
      return;
    }
    if (nr > 0)
      cta_gemm_fullk(nr, k, k, alpha, ta ? A + r0 : A + r0 * k, k, ta, Bm, k, beta, C0 ? C0 + r0 * k : nullptr, k,
                     C + r0 * k, k, sm);
  };
  // two products with the same B (row blocks of C = alpha op(A) B + beta C0 and C2 = alpha2 op(A2) B + beta2 C02):
  // B staged once for both, and twice the output tiles to spread over the warps
  auto rgemm2 = [&](const double* Bm, bool ta, double alpha, const double* A, double beta, const double* C0, double* C,
                    double alpha2, const double* A2, double beta2, const double* C02, double* C2) {
    if (SMALL || per > 16) {
      rgemm(alpha, A, ta, Bm, beta, C0, C);
      rgemm(alpha2, A2, ta, Bm, beta2, C02, C2);
      return;
    }
    if (nr > 0)
      cta_gemm_fullk(nr, k, k, alpha, ta ? A + r0 : A + r0 * k, k, ta, Bm, k, beta, C0 ? C0 + r0 * k : nullptr, k,
                     C + r0 * k, k, sm, ta ? A2 + r0 : A2 + r0 * k, alpha2, beta2, C02 ? C02 + r0 * k : nullptr,
                     C2 + r0 * k);
  };
  if (tid == 0) {
    s_hits = 0;
    g_fk_bulk = !SMALL && !ws.fk_nobulk && k > 64;   // (k = 64: cp.async staging measured faster, 60.8 vs 65.4 us)
    g_fk_phase = 0;
    if (!SMALL) {
      mbar_init(&g_fk_mbar, 1);
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
  }
  if (!SMALL) __syncthreads();
  if (crank == 0) RF_TSTAMP(ws, 20);
  if (ws.tlog && tid == 0 && crank == 0) g_gemm_tlog = ws.tlog + 40;
  if (ws.tlog && tid == 0 && crank == 0) g_fullk_tlog = g_fullk_tlog_first = ws.tlog + 56;
  if (ws.multi) {   // [M2 | G2 | rr2] of every rank, summed in rank order (M2, G2, rr2 are contiguous)
    const int64_t cnt = 2 * kk + k;
    for (int64_t e = crank * nt + tid; e < cnt; e += (int64_t)ncl * nt) {
      double sum = ws.mg_all[e];
      for (int r = 1; r < ws.world; ++r) sum += ws.mg_all[(int64_t)r * cnt + e];
      ws.M2[e] = sum;
    }
    cluster_sync();
  if (crank == 0) RF_TSTAMP(ws, 21);
  }
  if (SMALL) {   // every global input of the chain into shared memory in one round trip
    for (int e = tid; e < kk; e += nt) {
      cp_async8(S + 16 * kk + e, ws.L + e, true);
      cp_async8(S + 17 * kk + e, ws.T + e, true);
      cp_async8(Xp + e, Xtop + e, true);
      cp_async8(R1 + e, Wtop + e, true);
      cp_async8(Mp + e, ws.M2 + e, true);
      cp_async8(Gp + e, ws.G2 + e, true);
      cp_async8(Ui + e, ws.Uinv + e, true);
    }
    for (int j = tid; j < k; j += nt) {
      cp_async8(vec + j, ws.sigma + j, true);
      cp_async8(vec + k + j, ws.d + j, true);
      cp_async8(vec + 2 * k + j, ws.alpha + j, true);
      cp_async8(vec + 3 * k + j, ws.rr2 + j, true);
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
  }
  // (SMALL: in place on the shared copies; each element is read and written by one thread)
  const double* srcX = SMALL ? Xp : Xtop;
  const double* srcW = SMALL ? R1 : Wtop;
  const double* srcM = SMALL ? Mp : ws.M2;
  const double* srcG = SMALL ? Gp : ws.G2;
  const double* srcU = SMALL ? Ui : ws.Uinv;
  if (crank == 0) RF_TSTAMP(ws, 35);
  for (int i = r0 + (tid >> 5); i < r1; i += 32)
#pragma unroll 1
    for (int j = tid & 31; j < k; j += 32) {
    const int e = i * k + j;
    const double xp = srcX[e] * sig[j];
    const double w = srcW[e];
    Xp[e] = xp;
    R1[e] = fma(-xp, d[j], w * sig[j]);
    Mp[e] = sig[i] * srcM[e] * sig[j];
    Gp[e] = sig[i] * srcG[e] * sig[j];
    Ui[e] = sig[i] * srcU[e];                         // U'^{-1} = Sigma U^{-1}
  }
  if (crank == 0) RF_TSTAMP(ws, 36);
  cluster_sync();
  if (crank == 0) RF_TSTAMP(ws, 22);
  if (useH) {   // one stage instead of three (the T products were done by kxk_lu)
    // V_1 = R_1 - H1^T R_1 - H3^T M',  P~ = H2^T R_1 + H4^T M'  (each B staged once for two products)
    rgemm2(R1, true, -1.0, H, 1.0, R1, V1, 1.0, H + kk, 0.0, nullptr, Pt);
    rgemm2(Mp, true, -1.0, H + 2 * kk, 1.0, V1, V1, 1.0, H + 3 * kk, 1.0, Pt, Pt);
    if (crank == 0) RF_TSTAMP(ws, 23);
    if (crank == 0) RF_TSTAMP(ws, 24);
  } else {
  rgemm(1.0, Lm, true, R1, 0.0, nullptr, Z);        // Z = L^T R_1
  rgemm(1.0, Ui, true, Mp, 1.0, Z, Z);                //   + U'^{-T} M'
  cluster_sync();
  if (crank == 0) RF_TSTAMP(ws, 23);
  rgemm(1.0, Tm, true, Z, 0.0, nullptr, P);         // P = T^T Z
  cluster_sync();
  if (crank == 0) RF_TSTAMP(ws, 24);
  rgemm(-1.0, Lm, false, P, 1.0, R1, V1);           // V_1 = R_1 - L P
  rgemm(1.0, Ui, false, P, 0.0, nullptr, Pt);         // P~ = U'^{-1} P
  }
  // E_11 (line 6): beta needs the Gram G = X'^T X' = X'_1^T X'_1 + G'
  for (int i = r0 + (tid >> 5); i < r1; i += 32)
#pragma unroll 1
    for (int j = tid & 31; j < k; j += 32) {
    const int e = i * k + j;
    double v;
    if (ws.top_zero) {                                 // after Rayleigh-Ritz
      v = 0.0;
    } else if (i == j) {
      v = (1.0 - alp[i]) / 2.0;
    } else {
      const double gap = d[j] - d[i];
      if (fabs(gap) <= ws.delta) {
        atomicAdd(&s_hits, 1);
        double gsum = Gp[e];
        for (int l = 0; l < k; ++l) gsum = fma(Xp[l * k + i], Xp[l * k + j], gsum);
        v = ws.beta_zero ? 0.0 : -gsum / 2.0;
      } else {
        v = V1[e] / gap;
      }
    }
    E11[e] = v;
  }
  cluster_sync();
  if (crank == 0) RF_TSTAMP(ws, 25);
  rgemm(1.0, Gp, false, Pt, 0.0, nullptr, GPt);       // G' P~
  for (int i = r0 + (tid >> 5); i < r1; i += 32)
#pragma unroll 1
    for (int j = tid & 31; j < k; j += 32) S2[i * k + j] = (Mp[i * k + j] - GPt[i * k + j]) / d[j];
  cluster_sync();
  if (crank == 0) RF_TSTAMP(ws, 26);
  if (useH) {   // L B and U'^{-1} B directly (one stage instead of three)
    // L B = H1 E_11 + H2 S2,  U'^{-1} B = H3 E_11 + H4 S2
    rgemm2(E11, false, 1.0, H, 0.0, nullptr, LB, 1.0, H + 2 * kk, 0.0, nullptr, UB);
    rgemm2(S2, false, 1.0, H + kk, 1.0, LB, LB, 1.0, H + 3 * kk, 1.0, UB, UB);
    if (crank == 0) RF_TSTAMP(ws, 27);
    if (crank == 0) RF_TSTAMP(ws, 28);
  } else {
  rgemm(1.0, Lm, true, E11, 0.0, nullptr, Qm);   // Qm = L^T E_11
  rgemm(1.0, Ui, true, S2, 1.0, Qm, Qm);              //   + U'^{-T} S2
  cluster_sync();
  if (crank == 0) RF_TSTAMP(ws, 27);
  rgemm(1.0, Tm, false, Qm, 0.0, nullptr, B);       // B = T Qm
  cluster_sync();
  if (crank == 0) RF_TSTAMP(ws, 28);
  rgemm(1.0, Lm, false, B, 0.0, nullptr, LB);       // L B
  rgemm(1.0, Ui, false, B, 0.0, nullptr, UB);         // U'^{-1} B
  }
  // S7 folded into this kernel: the column norms of X~ over the
  // rows >= top follow from the pass-B sums, with x~_i = w'_i D^-1 - x'_i C' and w' = r' + x' D:
  //   ||x~_2j||^2 = (rr_j + 2 d_j M'_jj + d_j^2 G'_jj) / d_j^2 - (2 / d_j) sum_l C'_lj (M'_lj + d_j G'_lj)
  //                 + (C'^T G' C')_jj
  // (the first term ~ 1, the others O(residual): no cancellation).  1 / ||x~_j|| is then folded
  // into the top rows written here and into pass C's Csig and scal, so pass C writes the final X.
  double* Cp = S + 15 * kk;                            // C' = P~ D^-1 + U'^-1 B
  double* GC = Z;                                      // G' C' (Z is dead)
  for (int l = r0 + (tid >> 5); l < r1; l += 32)
#pragma unroll 1
    for (int j = tid & 31; j < k; j += 32) {
    const int e = l * k + j;
    Xt1[e] = Xp[e] + (E11[e] - LB[e]);                 // X~_1 = X'_1 + (E_11 - L B)  (top rows of X~)
    Cp[e] = Pt[e] / d[j] + UB[e];
    ws.Csig[e] = sig[l] * Cp[e];                       // Csig = Sigma (P~ D^{-1} + U'^{-1} B)
  }
  if (tid == 0) part[crank] = (double)s_hits;
  cluster_sync();
  if (crank == 0) RF_TSTAMP(ws, 29);
  rgemm(1.0, Gp, false, Cp, 0.0, nullptr, GC);
  // Gram deviation of the sweep's input (reorthogonalisation policy): G = X'_1^T X'_1 + G'
  if (ws.want_gram) {
    rgemm(1.0, Xp, true, Xp, 1.0, Gp, LB);
    double m = 0.0;
    for (int e = r0 * k + tid; e < r1 * k; e += nt) m = fmax(m, fabs(LB[e] - ((e / k == e % k) ? 1.0 : 0.0)));
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((tid & 31) == 0) s_red[0][tid >> 5] = m;
    __syncthreads();
    if (tid == 0) {
      for (int w = 1; w < nt / 32; ++w) m = fmax(m, s_red[0][w]);
      part[16 + crank] = m;
    }
  }
  constexpr int NQ = 7;
  // clustered: each CTA sums the NQ per-column quantities over its own rows (fixed row order) into its
  // slot of csp [ncl][NQ][k]; CTA 0 combines the slots in CTA order below (was: CTA 0 alone over all k
  // rows, 7.7 us at k = 128)
  double* csp = S + (KXK_SCRATCH_MATS - 2) * kk;       // 2 k^2 >= NQ ncl k for the cluster sizes used
  if (!SMALL) {
    double* qs = sm;                                   // [NQ][nr][k] (the product staging space is free)
    for (int e = tid; e < nr * k; e += nt) {
      const int r = e / k, j = e - r * k, ee = (r0 + r) * k + j;
      const double dj = d[j];
      const double x = Xt1[ee], rv = R1[ee], ev = E11[ee], pt = Pt[ee], c = Cp[ee];
      double* q = qs + (size_t)r * k + j;
      const size_t st = (size_t)nr * k;
      q[0] = x * x;                                    // ||x~_1j||^2 (top rows)
      q[st] = rv * rv;                                 // ||R_1j||^2
      q[2 * st] = ev * ev;                             // ||E_11 j||^2
      q[3 * st] = pt * Mp[ee];                         // (P~^T M')_jj
      q[4 * st] = pt * GPt[ee];                        // (P~^T G' P~)_jj
      q[5 * st] = c * fma(dj, Gp[ee], Mp[ee]);         // sum_l C'_lj (M'_lj + d_j G'_lj)
      q[6 * st] = c * GC[ee];                          // (C'^T G' C')_jj
    }
    __syncthreads();
    for (int t = tid; t < NQ * k; t += nt) {
      const int u = t / k, j = t - u * k;
      double a = 0.0;
      for (int r = 0; r < nr; ++r) a += qs[((size_t)u * nr + r) * k + j];
      csp[((size_t)crank * NQ + u) * k + j] = a;
    }
  }
  cluster_sync();
  if (crank == 0) RF_TSTAMP(ws, 30);
  if (crank == 0) {
    // SMALL: per-column sums over the k rows, by all 1024 threads: thread (g, j) takes rows l = g, g + NG, ..
    // (fixed partition, groups combined in order -- deterministic); clustered: the CTAs' slots
    const int NG = SMALL ? min(8, k) : ncl;            // partial groups (SMALL: a short combine chain)
    double* cs = cs_base;                              // [NG][NQ][k] partials (clustered: the slots, copied in)
    double* sd = cs_base + (size_t)(SMALL ? 8 : ncl) * NQ * k;   // d
    for (int j = tid; j < k; j += nt) sd[j] = d[j];
    if (!SMALL)   // one L2 round trip for all slots (combining straight from global cost ~7 us at k = 128)
      for (int e = tid; e < ncl * NQ * k; e += nt) cs[e] = csp[e];
    if (SMALL && tid < NG * k) {
      const int g = tid / k, j = tid % k;
      const double dj = d[j];
      double q[NQ] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll 1
      for (int l = g; l < k; l += NG) {
        const int e = l * k + j;
        const double x = Xt1[e], r = R1[e], ee = E11[e], pt = Pt[e], c = Cp[e];
        q[0] = fma(x, x, q[0]);                        // ||x~_1j||^2 (top rows)
        q[1] = fma(r, r, q[1]);                        // ||R_1j||^2
        q[2] = fma(ee, ee, q[2]);                      // ||E_11 j||^2
        q[3] = fma(pt, Mp[e], q[3]);                   // (P~^T M')_jj
        q[4] = fma(pt, GPt[e], q[4]);                  // (P~^T G' P~)_jj
        q[5] = fma(c, fma(dj, Gp[e], Mp[e]), q[5]);    // sum_l C'_lj (M'_lj + d_j G'_lj)
        q[6] = fma(c, GC[e], q[6]);                    // (C'^T G' C')_jj
      }
#pragma unroll
      for (int u = 0; u < NQ; ++u) cs[((size_t)g * NQ + u) * k + j] = q[u];
    }
    __syncthreads();
    {   // min_j |d_j - d_i| over i != j: 8 lanes per column, each over every 8th i, then a min over the lanes
      const int j = tid >> 3, sl = tid & 7;
      double mg = INFINITY;
      if (j < k)
#pragma unroll 1
        for (int i = sl; i < k; i += 8)
          if (i != j) mg = fmin(mg, fabs(sd[j] - sd[i]));
      for (int o = 1; o < 8; o <<= 1) mg = fmin(mg, __shfl_xor_sync(0xffffffffu, mg, o));
      if (j < k && sl == 0) s_red[2][j] = mg;
    }
    RF_TSTAMP(ws, 33);
    if (tid < k) {
      const int j = tid;
      double q[NQ];
#pragma unroll
      for (int u = 0; u < NQ; ++u) {
        q[u] = cs[(size_t)u * k + j];
#pragma unroll 1
        for (int g = 1; g < NG; ++g) q[u] += cs[((size_t)g * NQ + u) * k + j];
      }
      const double nt2 = q[0];
      ws.ntop[j] = nt2;
      const double e2 = (rr2p[j] - 2.0 * q[3] + q[4]) / (d[j] * d[j]);
      s_red[0][j] = q[1] + rr2p[j];
      s_red[1][j] = (ws.kjudge > 0 && j >= ws.kjudge) ? 0.0 : q[2] + e2;   // K > k: judge the leading kjudge
      s_red[3][j] = (sig[j] < 0.0) ? 1.0 : 0.0;
      // column norm of X~: top rows + the identity above -> 1 / ||x~_j||
      const double dj = sd[j];
      const double t1 = fma(dj, fma(dj, Gp[j * k + j], 2.0 * Mp[j * k + j]), rr2p[j]) / (dj * dj);
      const double tail = t1 - 2.0 * q[5] / dj + q[6];
      const double nrm = sqrt(nt2 + tail);
      const double inv = ws.normalize ? 1.0 / nrm : 1.0;
      if (!isfinite(inv) || !(nrm > 0.0)) atomicCAS(ws.status, ST_OK, ST_DIVERGED);
      ws.invn[j] = inv;
      ws.scal[j] = sig[j] / d[j] * inv;
    }
    __syncthreads();
    RF_TSTAMP(ws, 34);
    if (tid < 32) {   // warp 0: lane sums over j = lane, lane + 32, .., then a xor butterfly (every lane equal)
      double rr = 0.0, en = 0.0, mg = INFINITY, fl = 0.0, hits = 0.0, gmax = -1.0;
#pragma unroll 1
      for (int j = tid; j < k; j += 32) { rr += s_red[0][j]; en += s_red[1][j]; mg = fmin(mg, s_red[2][j]); fl += s_red[3][j]; }
      for (int o = 16; o > 0; o >>= 1) {
        rr += __shfl_xor_sync(0xffffffffu, rr, o);
        en += __shfl_xor_sync(0xffffffffu, en, o);
        mg = fmin(mg, __shfl_xor_sync(0xffffffffu, mg, o));
        fl += __shfl_xor_sync(0xffffffffu, fl, o);
      }
      if (tid == 0)
      for (int c = 0; c < ncl; ++c) {
        hits += part[c];
        if (ws.want_gram) gmax = fmax(gmax, part[16 + c]);
      }
      if (tid == 0) {
      ws.stats[0] = sqrt(rr) / ws.normA;
      ws.stats[1] = sqrt(fmax(en, 0.0));
      ws.stats[2] = (k > 1) ? mg : 0.0;
      ws.stats[3] = hits;
      ws.stats[4] = (fl > 0.0) ? 1.0 : 0.0;
      ws.stats[5] = rr;
      ws.stats[6] = ws.want_gram ? gmax : -1.0;
      }
    }
  }
  cluster_sync();
  if (crank == 0) RF_TSTAMP(ws, 31);
  for (int i = r0 + (tid >> 5); i < r1; i += 32)
#pragma unroll 1
    for (int j = tid & 31; j < k; j += 32) {
    const int e = i * k + j;
    const double inv = ws.invn[j];
    Xtop[e] = Xt1[e] * inv;                            // final top rows of X
    ws.Csig[e] *= inv;
    if (SMALL) { ws.E11[e] = E11[e]; ws.Xt[e] = Xt1[e]; }   // (the global copies: debug / Rayleigh-Ritz readers)
  }
  if (crank == 0) RF_TSTAMP(ws, 32);
}
template <bool SMALL>
__global__ void __launch_bounds__(KXK_THREADS) kxk_finish_kernel(Ws ws, double* __restrict__ Xtop,
                                                                 const double* __restrict__ Wtop) {
  extern __shared__ __align__(16) double sm[];
  __shared__ int s_hits;
  __shared__ double s_red[4][KMAX];
  griddep_wait();   // (programmatic dependent launch: the predecessor's writes are visible after this)
  if (*ws.status != ST_OK) return;
  kxk_finish_body<SMALL>(ws, Xtop, Wtop, sm, s_hits, s_red);
}

// ---------------------------------------------------------------- rr_kxk (Rayleigh-Ritz, Sec. 3.4)
// (X^T A X) S = (X^T X) S D~,  Z = X S  (Z^T Z = I, Z^T A Z = D~).  Inputs: the
// pass-B sums over rows >= top with D = 0, M2 = X_2^T W_2 and G2 = X_2^T X_2, plus the top rows.
//   M = M2 + X_1^T W_1, G = G2 + X_1^T X_1;  M <- (M + M^T)/2                      (reading RR1)
//   G = L L^T (Cholesky);  Ui = L^{-T};  C = Ui^T M Ui;  C = Q diag(d) Q^T by parallel Jacobi
//   (round-robin pairs, k/2 disjoint rotations per step, until off(C) <= (u ||C||_F)^2)   (RR2)
//   Ritz pairs by descending d; each Q column signed so its largest |entry| is positive  (RR3)
//   S = Ui Q;  top rows Z_1 = X_1 S -> X~;  Csig = -S, scal = 0 so that pass C forms Z_2 = X_2 S.
__device__ void rr_rotate(int k, double* C, double* Q, int m, int round, double* cs, double* sn, int* pp,
                          int* qq) {
  const int tid = threadIdx.x, npair = m / 2;
  if (tid < npair) {   // round-robin pairing of players 0..m-1 (player 0 fixed)
    auto player = [&](int j) { return j == 0 ? 0 : 1 + (j - 1 + round) % (m - 1); };
    int p = player(tid), q = player(m - 1 - tid);
    if (p > q) { const int t = p; p = q; q = t; }
    double c = 1.0, s = 0.0;
    if (q < k) {
      const double apq = C[p * k + q];
      if (apq != 0.0) {
        const double theta = (C[q * k + q] - C[p * k + p]) / (2.0 * apq);
        const double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        c = 1.0 / sqrt(t * t + 1.0);
        s = t * c;
      }
    }
    cs[tid] = c; sn[tid] = s; pp[tid] = p; qq[tid] = q;
  }
  __syncthreads();
  for (int e = tid; e < k * npair; e += KXK_THREADS) {   // C <- C J, Q <- Q J (columns p, q)
    const int t = e % npair, r = e / npair, p = pp[t], q = qq[t];
    if (q >= k) continue;
    const double c = cs[t], s = sn[t];
    const double cp = C[r * k + p], cq = C[r * k + q];
    C[r * k + p] = c * cp - s * cq;
    C[r * k + q] = s * cp + c * cq;
    const double qp = Q[r * k + p], qv = Q[r * k + q];
    Q[r * k + p] = c * qp - s * qv;
    Q[r * k + q] = s * qp + c * qv;
  }
  __syncthreads();
  for (int e = tid; e < k * npair; e += KXK_THREADS) {   // C <- J^T C (rows p, q)
    const int t = e % npair, r = e / npair, p = pp[t], q = qq[t];
    if (q >= k) continue;
    const double c = cs[t], s = sn[t];
    const double cp = C[p * k + r], cq = C[q * k + r];
    C[p * k + r] = c * cp - s * cq;
    C[q * k + r] = s * cp + c * cq;
  }
  __syncthreads();
}

// mode 1: reorthogonalisation by Cholesky QR: S = L^{-T} (no pencil, no Jacobi), and
// max |X^T X - I| before it into ritz[0].
__global__ void __launch_bounds__(KXK_THREADS) rr_kxk_kernel(Ws ws, const double* __restrict__ Xtop,
                                                             const double* __restrict__ Wtop, int mode) {
  extern __shared__ __align__(16) double sm[];
  __shared__ double s_cs[KMAX / 2 + 1], s_sn[KMAX / 2 + 1], s_red[KXK_THREADS / 32];
  __shared__ int s_p[KMAX / 2 + 1], s_q[KMAX / 2 + 1], s_ord[KMAX], s_bad;
  __shared__ double s_d[KMAX];
  griddep_wait();   // (programmatic dependent launch: the predecessor's writes are visible after this)
  if (*ws.status != ST_OK) return;
  const int k = ws.k, kk = k * k, tid = threadIdx.x, nt = KXK_THREADS;
  double* S = ws.scratch;
  double *M = S, *G = S + kk, *Lt = S + 2 * kk, *Ui = S + 3 * kk, *T1 = S + 4 * kk, *Cm = S + 5 * kk,
         *Q = S + 6 * kk, *Qs = S + 7 * kk, *Sm = S + 8 * kk, *tmp = S + 9 * kk, *X1 = S + 10 * kk;
  if (tid == 0) s_bad = 0;
  if (ws.multi) {   // [M2 | G2 | rr2] of every rank, summed in rank order
    const int64_t cnt = 2 * kk + k;
    for (int64_t e = tid; e < cnt; e += nt) {
      double sum = ws.mg_all[e];
      for (int r = 1; r < ws.world; ++r) sum += ws.mg_all[(int64_t)r * cnt + e];
      ws.M2[e] = sum;
    }
  }
  for (int e = tid; e < kk; e += nt) X1[e] = Xtop[e];
  __syncthreads();
  if (mode == 0)
    cta_gemm(k, k, k, 1.0, X1, k, true, Wtop, k, false, 1.0, ws.M2, k, M, k, sm);   // M = M2 + X_1^T W_1
  cta_gemm(k, k, k, 1.0, X1, k, true, X1, k, false, 1.0, ws.G2, k, G, k, sm);      // G = G2 + X_1^T X_1
  if (mode == 0) {
    for (int e = tid; e < kk; e += nt) {                                            // RR1
      const int i = e / k, j = e % k;
      if (i < j) { const double m = (M[e] + M[j * k + i]) / 2.0; M[e] = m; M[j * k + i] = m; }
    }
  } else {                                                                          // Gram deviation
    double gm = 0.0;
    for (int e = tid; e < kk; e += nt) gm = fmax(gm, fabs(G[e] - ((e / k == e % k) ? 1.0 : 0.0)));
    for (int o = 16; o > 0; o >>= 1) gm = fmax(gm, __shfl_xor_sync(0xffffffffu, gm, o));
    if ((tid & 31) == 0) s_red[tid >> 5] = gm;
    __syncthreads();
    if (tid == 0) {
      for (int w = 1; w < nt / 32; ++w) gm = fmax(gm, s_red[w]);
      ws.ritz[0] = gm;
    }
  }
  __syncthreads();
  // Cholesky G = L L^T, right-looking, L in G's lower triangle
  if (tid < k) s_d[tid] = G[tid * k + tid];   // original diagonal (singularity threshold)
  __syncthreads();
  for (int j = 0; j < k; ++j) {
    if (tid == 0) {
      const double g = G[j * k + j];
      if (!(g > 4.0 * k * 1.1102230246251565e-16 * s_d[j])) s_bad = 1;   // X rank deficient (RR2)
      G[j * k + j] = sqrt(fmax(g, 0.0));
    }
    __syncthreads();
    if (s_bad) break;
    const double ljj = G[j * k + j];
    for (int i = j + 1 + tid; i < k; i += nt) G[i * k + j] /= ljj;
    __syncthreads();
    for (int e = tid; e < (k - j - 1) * (k - j - 1); e += nt) {
      const int a = j + 1 + e / (k - j - 1), b = j + 1 + e % (k - j - 1);
      if (b <= a) G[a * k + b] -= G[a * k + j] * G[b * k + j];
    }
    __syncthreads();
  }
  if (s_bad) {
    if (tid == 0) atomicCAS(ws.status, ST_OK, ST_E_INVALID);   // X^T X not positive definite
    return;
  }
  for (int e = tid; e < kk; e += nt) {   // Lt = L^T (upper, non-unit)
    const int i = e / k, j = e % k;
    Lt[e] = (j >= i) ? G[j * k + i] : 0.0;
  }
  __syncthreads();
  cta_trinv(k, Lt, true, Ui, tmp, sm);                                            // Ui = L^{-T}
  if (mode == 1) {                                                                // Cholesky QR: S = L^{-T}
    cta_gemm(k, k, k, 1.0, X1, k, false, Ui, k, false, 0.0, nullptr, 0, ws.Xt, k, sm);  // Z_1 = X_1 S
    for (int e = tid; e < kk; e += nt) ws.Csig[e] = -Ui[e];
    if (tid < k) {
      ws.scal[tid] = 0.0;
      double nt2 = 0.0;
      for (int i = 0; i < k; ++i) nt2 = fma(ws.Xt[i * k + tid], ws.Xt[i * k + tid], nt2);
      ws.ntop[tid] = nt2;
    }
    return;
  }
  cta_gemm(k, k, k, 1.0, Ui, k, true, M, k, false, 0.0, nullptr, 0, T1, k, sm);   // Ui^T M
  cta_gemm(k, k, k, 1.0, T1, k, false, Ui, k, false, 0.0, nullptr, 0, Cm, k, sm); // C = Ui^T M Ui
  for (int e = tid; e < kk; e += nt) {
    const int i = e / k, j = e % k;
    Q[e] = (i == j) ? 1.0 : 0.0;
    if (i < j) { const double m = (Cm[e] + Cm[j * k + i]) / 2.0; Cm[e] = m; Cm[j * k + i] = m; }
  }
  __syncthreads();
  // parallel Jacobi sweeps (RR2)
  const int m = (k + 1) & ~1;
  const double u = 1.1102230246251565e-16;
  for (int sweep = 0; sweep < 60; ++sweep) {
    double off = 0.0, fro = 0.0;
    for (int e = tid; e < kk; e += nt) {
      const double v = Cm[e];
      fro += v * v;
      if (e / k != e % k) off += v * v;
    }
    for (int o = 16; o > 0; o >>= 1) { off += __shfl_xor_sync(0xffffffffu, off, o); fro += __shfl_xor_sync(0xffffffffu, fro, o); }
    __shared__ double s_off[KXK_THREADS / 32];
    if ((tid & 31) == 0) { s_off[tid >> 5] = off; s_red[tid >> 5] = fro; }
    __syncthreads();
    if (tid == 0) {
      double a = 0.0, b = 0.0;
      for (int w = 0; w < nt / 32; ++w) { a += s_off[w]; b += s_red[w]; }
      s_off[0] = a; s_red[0] = b;
    }
    __syncthreads();
    const bool done = s_off[0] <= u * u * s_red[0];
    __syncthreads();
    if (done || k == 1) break;
    for (int round = 0; round < m - 1; ++round) rr_rotate(k, Cm, Q, m, round, s_cs, s_sn, s_p, s_q);
  }
  // RR3: descending Ritz values (stable), columns signed by their largest |entry|
  if (tid < k) s_d[tid] = Cm[tid * k + tid];
  __syncthreads();
  if (tid == 0) {
    for (int j = 0; j < k; ++j) s_ord[j] = j;
    for (int a = 1; a < k; ++a) {
      const int v = s_ord[a];
      int b = a - 1;
      while (b >= 0 && s_d[s_ord[b]] < s_d[v]) { s_ord[b + 1] = s_ord[b]; --b; }
      s_ord[b + 1] = v;
    }
  }
  __syncthreads();
  if (tid < k) {
    const int j = tid, o = s_ord[j];
    int im = 0;
    for (int i = 1; i < k; ++i)
      if (fabs(Q[i * k + o]) > fabs(Q[im * k + o])) im = i;
    const double sg = (Q[im * k + o] < 0.0) ? -1.0 : 1.0;
    for (int i = 0; i < k; ++i) Qs[i * k + j] = sg * Q[i * k + o];
    ws.ritz[j] = s_d[o];
  }
  __syncthreads();
  cta_gemm(k, k, k, 1.0, Ui, k, false, Qs, k, false, 0.0, nullptr, 0, Sm, k, sm);   // S = Ui Q
  cta_gemm(k, k, k, 1.0, X1, k, false, Sm, k, false, 0.0, nullptr, 0, ws.Xt, k, sm);  // Z_1 = X_1 S
  for (int e = tid; e < kk; e += nt) ws.Csig[e] = -Sm[e];                         // pass C: Z_2 = X_2 S
  if (tid < k) {
    ws.scal[tid] = 0.0;
    double nt2 = 0.0;
    for (int i = 0; i < k; ++i) nt2 = fma(ws.Xt[i * k + tid], ws.Xt[i * k + tid], nt2);
    ws.ntop[tid] = nt2;
  }
}

// ---------------------------------------------------------------- norm_reduce
// Column sums of x~^2 over pass C's slots: P = 1024 / k contiguous slot ranges per column summed
// in parallel (loads batched 8 at a time), then a fixed pairwise tree over the ranges, plus the
// top block (deterministic; was one thread per column, latency bound at ~40 us for 444 slots).
__global__ void __launch_bounds__(KXK_THREADS) norm_reduce_kernel(Ws ws) {
  __shared__ double part[KXK_THREADS];
  griddep_wait();   // (programmatic dependent launch: the predecessor's writes are visible after this)
  if (*ws.status != ST_OK) return;
  const int k = ws.k, tid = threadIdx.x;
  const int P = KXK_THREADS / k, j = tid % k, p = tid / k;
  double s = 0.0;
  if (p < P) {
    const int q0 = (int)((int64_t)ws.n_nslot * p / P), q1 = (int)((int64_t)ws.n_nslot * (p + 1) / P);
    int q = q0;
    for (; q + 8 <= q1; q += 8) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = ws.nslot[(int64_t)(q + u) * ws.kp + j];
#pragma unroll
      for (int u = 0; u < 8; ++u) s += v[u];
    }
    for (; q < q1; ++q) s += ws.nslot[(int64_t)q * ws.kp + j];
  }
  part[tid] = s;
  __syncthreads();
  for (int st = 1; st < P; st *= 2) {
    if (p < P && (p % (2 * st)) == 0 && p + st < P) part[tid] += part[tid + st * k];
    __syncthreads();
  }
  if (tid >= k) return;
  s = ws.ntop[j] + part[j];
  if (ws.multi) {          // partial for the all-gather; normalize_kernel combines in rank order
    ws.nrm_send[j] = s;
    return;
  }
  const double nrm = sqrt(s);
  ws.invn[j] = 1.0 / nrm;
  if (!isfinite(ws.invn[j]) || !(nrm > 0.0)) atomicCAS(ws.status, ST_OK, ST_DIVERGED);
}

// ---------------------------------------------------------------- debug: materialise Y
// Y (in: X^ of the sweep, out: Y): rows < top -> L; rows >= top: y_i U = x_i (forward
// substitution, ascending h) -- the tall-skinny triangular apply Y_2 = X^_2 U^{-1}.
__global__ void trsm_y_kernel(Ws ws, double* __restrict__ Y) {
  const int k = ws.k;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ws.n_loc;
       i += (int64_t)gridDim.x * blockDim.x) {
    double* y = Y + i * k;
    if (i < ws.top) {
      for (int h = 0; h < k; ++h) y[h] = ws.L[i * k + h];
    } else {
      for (int h = 0; h < k; ++h) {
        double s = y[h];
        for (int l = 0; l < h; ++l) s = __dadd_rn(s, -__dmul_rn(y[l], ws.U[l * k + h]));
        y[h] = __ddiv_rn(s, ws.U[h * k + h]);
      }
    }
  }
}

}  // namespace rf
