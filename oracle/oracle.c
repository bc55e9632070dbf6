/*
 * oracle/oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, literal CPU FP64 implementation of one refinement sweep of
 * arXiv 2602.23778 ("iterative refinement for a subset of eigenvectors"),
 * written from PAPER.md and nothing else.  It shares no code, header, table or
 * constant generator with the CUDA path (paper_2602_23778_b200/csrc) and
 * neither side includes or imports the other.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.
 *
 * Citations are to /root/reference/PAPER.md lines (section / algorithm / eq.).
 *   Alg. 2  modified_LU         PAPER.md:271-284 (Sec. 3.1.1)
 *   Alg. 3  CompactWY_LU
 *   Alg. 1  CompactWY
 *   one-time X <- X*Sigma
 *   Alg. 4  the sweep
 *   eq. Rayleigh / Ediag / V-def / Eoffdiag
 *   beta choices
 *   implicit H B
 *   stopping criteria
 *   normalisation
 *   delta = c ||A|| u, c = 10
 *   shift B = A - alpha I       PAPER.md:1194-1209 (Sec. 5.1)
 *   Rayleigh-Ritz preprocessing PAPER.md:904-930 (Sec. 3.4), beta = 0 after it
 *   shift-and-square B = A^2 - alpha I, applied as A (A X)   PAPER.md:1218-1243 (Sec. 5.2)
 *   refine K > k columns, judge the leading k
 *
 * Readings where the paper is silent or misprinted are listed in DESIGN.md
 * ("Readings of the paper"); the ones that change arithmetic here:
 *   R1 sign(0) = +1 in Alg. 2 line 2.
 *   R2 Alg. 3's Ensure line holds as H I_{n,k} = Q Sigma (not Q); therefore the
 *      sweep applies the paper's sign transformation X <- X Sigma (and W <- W
 *      Sigma) right after building the WY factors, every sweep.
 *   R4 ||A|| in delta and in the relative residual is ||A - shift I||_inf.
 *   R5 the delta test is inclusive (|d_j - d_i| <= delta).
 *   R6 beta_ij = -x_i^T x_j / 2 by default, 0 under beta_zero.
 *   R7 columns are normalised (true division) at the end of every sweep.
 *
 * Precision: FP64 throughout.  Every length-n reduction is a
 * Neumaier-compensated sum in ascending row order; every product with A is an
 * fma chain in ascending column order.  k-length inner sums are plain FP64 in
 * loop order.  OpenMP only splits independent output entries, each of which is
 * computed start-to-finish by one thread in a fixed order, so the result does
 * not depend on the thread count.
 *
 * Layout: every n x k block is row-major with leading dimension k (entry (i,j)
 * at [i*k + j]); k x k blocks likewise.  Dense A is row-major with leading
 * dimension lda.  CSR A stores both triangles, int32 indices, sorted columns.
 *
 * Parity pins: see tests/test_oracle_*.py.  Functions with no independent pin
 * are marked "parity unpinned" below (only the beta/delta branch).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* status values of this oracle (the C-ABI defines its own; tests compare by value) */
enum {
  OR_OK = 0, OR_MAXITER = 1, OR_DIVERGED = 2,
  OR_E_INVALID = -1, OR_E_NEAR_ZERO_RQ = -2, OR_E_ZERO_PIVOT = -3, OR_E_NOMEM = -6
};

#define IDX(i, j, ld) ((int64_t)(i) * (int64_t)(ld) + (int64_t)(j))

/* ---- Neumaier compensated summation (used for every length-n reduction) ---- */
typedef struct { double s, c; } nsum;
static inline void nsum_add(nsum* a, double x) {
  double t = a->s + x;
  if (fabs(a->s) >= fabs(x)) a->c += (a->s - t) + x;
  else                       a->c += (x - t) + a->s;
  a->s = t;
}
static inline double nsum_val(const nsum* a) { return a->s + a->c; }

/* =========================================================================
 * The operator: A or A - shift*I (Alg. 4 line 1; Sec. 5.1
 * PAPER.md:1203 "B = A - alpha I").
 * ========================================================================= */
typedef struct {
  int is_csr;
  int64_t n;
  /* dense */
  const double* A; int64_t lda;
  /* csr */
  const int32_t* row_ptr; const int32_t* col_idx; const double* val;
  double shift;
  int square;   /* 1: the operator is A^2 - shift I (Sec. 5.2), applied as A (A X) */
} op_t;

/* W = A X  (no shift): fma chain over the row of A in ascending column order from 0. */
static void op_product(const op_t* op, int32_t k, const double* X, double* W) {
  const int64_t n = op->n;
  const int64_t RB = 8;   /* rows per block: cache reuse of X only, per-entry order unchanged */
  #pragma omp parallel for schedule(static)
  for (int64_t i0 = 0; i0 < n; i0 += RB) {
    const int64_t i1 = (i0 + RB < n) ? i0 + RB : n;
    for (int64_t i = i0; i < i1; ++i)
      for (int32_t j = 0; j < k; ++j) W[IDX(i, j, k)] = 0.0;
    if (op->is_csr) {
      for (int64_t i = i0; i < i1; ++i) {
        double* w = W + IDX(i, 0, k);
        for (int32_t p = op->row_ptr[i]; p < op->row_ptr[i + 1]; ++p) {
          const double a = op->val[p];
          const double* x = X + IDX(op->col_idx[p], 0, k);
          for (int32_t j = 0; j < k; ++j) w[j] = fma(a, x[j], w[j]);
        }
      }
    } else {
      for (int64_t l = 0; l < n; ++l) {
        const double* x = X + IDX(l, 0, k);
        for (int64_t i = i0; i < i1; ++i) {
          const double a = op->A[IDX(i, l, op->lda)];
          double* w = W + IDX(i, 0, k);
          for (int32_t j = 0; j < k; ++j) w[j] = fma(a, x[j], w[j]);
        }
      }
    }
  }
}

/* W = A X - shift X  (or A (A X) - shift X when square; A^2 is never formed):
 * each product an fma chain in ascending column order, then (shift != 0) w_ij = fma(-shift, x_ij, w_ij). */
static void op_apply(const op_t* op, int32_t k, const double* X, double* W) {
  const int64_t n = op->n;
  if (op->square) {
    double* T = (double*)malloc(sizeof(double) * (size_t)n * (size_t)k);
    op_product(op, k, X, T);
    op_product(op, k, T, W);
    free(T);
  } else {
    op_product(op, k, X, W);
  }
  if (op->shift != 0.0) {
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i)
      for (int32_t j = 0; j < k; ++j) W[IDX(i, j, k)] = fma(-op->shift, X[IDX(i, j, k)], W[IDX(i, j, k)]);
  }
}

/* ||A - shift I||_inf = max_i sum_l |a_il - shift delta_il|   (reading R4); for the squared
 * operator the bound ||A||_inf^2 + |shift| >= ||A^2 - shift I||_2 (reading SQ1: A^2 is never formed) */
static double op_norm_inf_plain(const op_t* op);
static double op_norm_inf(const op_t* op) {
  if (op->square) {
    op_t a = *op;
    a.square = 0; a.shift = 0.0;
    const double na = op_norm_inf_plain(&a);
    return na * na + fabs(op->shift);
  }
  return op_norm_inf_plain(op);
}
static double op_norm_inf_plain(const op_t* op) {
  double best = 0.0;
  for (int64_t i = 0; i < op->n; ++i) {
    nsum s = {0, 0};
    if (op->is_csr) {
      int diag_seen = 0;
      for (int32_t p = op->row_ptr[i]; p < op->row_ptr[i + 1]; ++p) {
        double a = op->val[p];
        if (op->col_idx[p] == i) { a -= op->shift; diag_seen = 1; }
        nsum_add(&s, fabs(a));
      }
      if (!diag_seen) nsum_add(&s, fabs(op->shift));
    } else {
      const double* arow = op->A + IDX(i, 0, op->lda);
      for (int64_t l = 0; l < op->n; ++l) nsum_add(&s, fabs(l == i ? arow[l] - op->shift : arow[l]));
    }
    double v = nsum_val(&s);
    if (v > best) best = v;
  }
  return best;
}

double oracle_norm_inf_dense(int64_t n, const double* A, int64_t lda, double shift) {
  op_t op = {0, n, A, lda, NULL, NULL, NULL, shift};
  return op_norm_inf(&op);
}
double oracle_norm_inf_csr(int64_t n, const int32_t* rp, const int32_t* ci, const double* v, double shift) {
  op_t op = {1, n, NULL, 0, rp, ci, v, shift};
  return op_norm_inf(&op);
}

int oracle_apply_dense(int64_t n, int32_t k, const double* A, int64_t lda, double shift,
                       const double* X, double* W) {
  op_t op = {0, n, A, lda, NULL, NULL, NULL, shift};
  op_apply(&op, k, X, W);
  return OR_OK;
}
int oracle_apply_csr(int64_t n, int32_t k, const int32_t* rp, const int32_t* ci, const double* v,
                     double shift, const double* X, double* W) {
  op_t op = {1, n, NULL, 0, rp, ci, v, shift};
  op_apply(&op, k, X, W);
  return OR_OK;
}

/* =========================================================================
 * Alg. 2  [Y,U,Sigma] = modified_LU(Q)
 *   for j = 1..k:
 *     sigma_j = -sign(q_jj)                   (R1: sign(0) = +1)
 *     q_jj    = q_jj - sigma_j
 *     q_lj    = q_lj / q_jj        (j+1 <= l <= n)
 *     q_lh    = q_lh - q_lj q_jh   (j+1 <= l <= n, j+1 <= h <= k)
 * In place on Q (n x k): the strict lower part becomes Y (unit diagonal
 * implied), the upper triangle of the top k x k block becomes U.
 * Returns OR_E_ZERO_PIVOT if a shifted pivot is exactly zero (cannot happen
 * for |sigma_j| = 1 unless q_jj = sigma_j exactly; defensive).
 * ========================================================================= */
int oracle_modified_lu(int64_t n, int32_t k, double* Q, double* sigma) {
  for (int32_t j = 0; j < k; ++j) {
    const double qjj = Q[IDX(j, j, k)];
    const double s = -(qjj >= 0.0 ? 1.0 : -1.0);   /* -sign(q_jj), sign(0)=+1 */
    sigma[j] = s;
    Q[IDX(j, j, k)] = qjj - s;
    const double piv = Q[IDX(j, j, k)];
    if (piv == 0.0) return OR_E_ZERO_PIVOT;
    #pragma omp parallel for schedule(static)
    for (int64_t l = j + 1; l < n; ++l) {
      double* ql = Q + IDX(l, 0, k);
      ql[j] = ql[j] / piv;
      const double qlj = ql[j];
      for (int32_t h = j + 1; h < k; ++h) ql[h] = ql[h] - qlj * Q[IDX(j, h, k)];
    }
  }
  return OR_OK;
}

/* Split the in-place result of Alg. 2 into explicit Y (n x k, unit lower
 * trapezoidal) and U (k x k upper). */
static void split_lu(int64_t n, int32_t k, const double* LU, double* Y, double* U) {
  for (int64_t i = 0; i < n; ++i)
    for (int32_t j = 0; j < k; ++j)
      Y[IDX(i, j, k)] = (i > j) ? LU[IDX(i, j, k)] : (i == j ? 1.0 : 0.0);
  if (U)
    for (int32_t i = 0; i < k; ++i)
      for (int32_t j = 0; j < k; ++j) U[IDX(i, j, k)] = (j >= i) ? LU[IDX(i, j, k)] : 0.0;
}

/* Solve T * L^T = B for T, L = Y_1 unit lower (k x k), i.e. T = B L^{-T}.
 * Row by row, ascending column:  t_ij = b_ij - sum_{l<j} t_il * L_jl. */
static void solve_right_unit_lower_transpose(int32_t k, const double* L, const double* B, double* T) {
  for (int32_t i = 0; i < k; ++i)
    for (int32_t j = 0; j < k; ++j) {
      double t = B[IDX(i, j, k)];
      for (int32_t l = 0; l < j; ++l) t -= T[IDX(i, l, k)] * L[IDX(j, l, k)];
      T[IDX(i, j, k)] = t;
    }
}

/* =========================================================================
 * Alg. 3  [Y,T,Sigma] = CompactWY_LU(Q)
 *   [Y,U,Sigma] = modified_LU(Q);  T = -U Sigma Y_1^{-T}
 * (Ensure line: H I_{n,k} = Q Sigma, reading R2.)
 * Q is not modified.  Y: n x k, T: k x k, sigma: k, U (optional): k x k.
 * ========================================================================= */
int oracle_compact_wy_lu(int64_t n, int32_t k, const double* Q, double* Y, double* T,
                         double* sigma, double* U_out) {
  double* LU = (double*)malloc(sizeof(double) * (size_t)n * (size_t)k);
  double* U = (double*)malloc(sizeof(double) * (size_t)k * (size_t)k);
  double* B = (double*)malloc(sizeof(double) * (size_t)k * (size_t)k);
  if (!LU || !U || !B) { free(LU); free(U); free(B); return OR_E_NOMEM; }
  memcpy(LU, Q, sizeof(double) * (size_t)n * (size_t)k);
  int st = oracle_modified_lu(n, k, LU, sigma);
  if (st == OR_OK) {
    split_lu(n, k, LU, Y, U);
    /* B = -U Sigma (column j of U scaled by sigma_j) */
    for (int32_t i = 0; i < k; ++i)
      for (int32_t j = 0; j < k; ++j) B[IDX(i, j, k)] = -(U[IDX(i, j, k)] * sigma[j]);
    solve_right_unit_lower_transpose(k, Y, B, T);  /* Y_1 = leading k x k block of Y */
    if (U_out) memcpy(U_out, U, sizeof(double) * (size_t)k * (size_t)k);
  }
  free(LU); free(U); free(B);
  return st;
}

/* =========================================================================
 * Alg. 1  [Y,T] = CompactWY(Q)
 *   Y = Q - I_{n,k};  T = -Y_1^{-T}
 * Y_1 is a general k x k matrix here; T = -Y_1^{-T} is computed by Gaussian
 * elimination with partial pivoting on Y_1^T X = -I.  Returns OR_E_ZERO_PIVOT
 * if Y_1 is exactly singular.  Used by the Alg. 1 == Alg. 3 pin only.
 * ========================================================================= */
int oracle_compact_wy(int64_t n, int32_t k, const double* Q, double* Y, double* T) {
  for (int64_t i = 0; i < n; ++i)
    for (int32_t j = 0; j < k; ++j) Y[IDX(i, j, k)] = Q[IDX(i, j, k)] - (i == j ? 1.0 : 0.0);
  /* M = Y_1^T (k x k), RHS = -I; solve M T = -I  => T = -Y_1^{-T} */
  double* M = (double*)malloc(sizeof(double) * (size_t)k * (size_t)k);
  if (!M) return OR_E_NOMEM;
  for (int32_t i = 0; i < k; ++i)
    for (int32_t j = 0; j < k; ++j) { M[IDX(i, j, k)] = Y[IDX(j, i, k)]; T[IDX(i, j, k)] = (i == j) ? -1.0 : 0.0; }
  for (int32_t c = 0; c < k; ++c) {
    int32_t p = c;
    for (int32_t r = c + 1; r < k; ++r) if (fabs(M[IDX(r, c, k)]) > fabs(M[IDX(p, c, k)])) p = r;
    if (M[IDX(p, c, k)] == 0.0) { free(M); return OR_E_ZERO_PIVOT; }
    if (p != c)
      for (int32_t j = 0; j < k; ++j) {
        double t = M[IDX(c, j, k)]; M[IDX(c, j, k)] = M[IDX(p, j, k)]; M[IDX(p, j, k)] = t;
        t = T[IDX(c, j, k)]; T[IDX(c, j, k)] = T[IDX(p, j, k)]; T[IDX(p, j, k)] = t;
      }
    for (int32_t r = c + 1; r < k; ++r) {
      const double f = M[IDX(r, c, k)] / M[IDX(c, c, k)];
      for (int32_t j = c; j < k; ++j) M[IDX(r, j, k)] -= f * M[IDX(c, j, k)];
      for (int32_t j = 0; j < k; ++j) T[IDX(r, j, k)] -= f * T[IDX(c, j, k)];
    }
  }
  for (int32_t c = k - 1; c >= 0; --c)
    for (int32_t j = 0; j < k; ++j) {
      double t = T[IDX(c, j, k)];
      for (int32_t l = c + 1; l < k; ++l) t -= M[IDX(c, l, k)] * T[IDX(l, j, k)];
      T[IDX(c, j, k)] = t / M[IDX(c, c, k)];
    }
  free(M);
  return OR_OK;
}

/* =========================================================================
 * Implicit products with H = I - Y T Y^T
 *   H B   = B - Y (T   (Y^T B))
 *   H^T B = B - Y (T^T (Y^T B))
 * B, out: n x m row-major.  Y^T B: Neumaier over n; k-length sums plain.
 * out may alias B.
 * ========================================================================= */
static void yt_b(int64_t n, int32_t k, const double* Y, int32_t m, const double* B, double* Z) {
  /* Z (k x m) = Y^T B; entry (a,c) is a compensated sum over i ascending.  Rows are
   * visited in chunks so all threads share the chunk in cache; each entry is owned
   * by one thread for the whole sum, so the order is fixed. */
  nsum* acc = (nsum*)calloc((size_t)k * (size_t)m, sizeof(nsum));
  const int64_t CH = 256;
  for (int64_t i0 = 0; i0 < n; i0 += CH) {
    const int64_t i1 = (i0 + CH < n) ? i0 + CH : n;
    #pragma omp parallel for schedule(static)
    for (int32_t a = 0; a < k; ++a) {
      nsum* row = acc + IDX(a, 0, m);
      for (int64_t i = i0; i < i1; ++i) {
        const double y = Y[IDX(i, a, k)];
        const double* b = B + IDX(i, 0, m);
        for (int32_t c = 0; c < m; ++c) nsum_add(&row[c], y * b[c]);
      }
    }
  }
  for (int32_t a = 0; a < k; ++a)
    for (int32_t c = 0; c < m; ++c) Z[IDX(a, c, m)] = nsum_val(&acc[IDX(a, c, m)]);
  free(acc);
}

int oracle_apply_h(int64_t n, int32_t k, const double* Y, const double* T, int32_t m,
                   const double* B, double* out, int transpose) {
  double* Z = (double*)malloc(sizeof(double) * (size_t)k * (size_t)m);
  double* P = (double*)malloc(sizeof(double) * (size_t)k * (size_t)m);
  if (!Z || !P) { free(Z); free(P); return OR_E_NOMEM; }
  yt_b(n, k, Y, m, B, Z);
  for (int32_t a = 0; a < k; ++a)
    for (int32_t c = 0; c < m; ++c) {
      double s = 0.0;
      for (int32_t l = 0; l < k; ++l) s += (transpose ? T[IDX(l, a, k)] : T[IDX(a, l, k)]) * Z[IDX(l, c, m)];
      P[IDX(a, c, m)] = s;
    }
  #pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i)
    for (int32_t c = 0; c < m; ++c) {
      double s = 0.0;
      for (int32_t l = 0; l < k; ++l) s += Y[IDX(i, l, k)] * P[IDX(l, c, m)];
      out[IDX(i, c, m)] = B[IDX(i, c, m)] - s;
    }
  free(Z); free(P);
  return OR_OK;
}

/* =========================================================================
 * Alg. 4 -- one refinement sweep
 * ========================================================================= */
typedef struct {
  double delta_c;      /* c in delta = c ||A|| u, default 10 */
  int32_t beta_zero;   /* 0: beta_ij = -x_i^T x_j / 2; 1: beta = 0 (:460) */
  int32_t normalize;   /* 1: normalise columns after the update */
  int32_t top_zero;    /* 1: E_11 = 0 -- the sweep follows Rayleigh-Ritz (reading RR4) */
  int32_t kjudge;      /* > 0: corr_norm over the leading kjudge columns only (K > k) */
  int32_t want_gram;   /* 1: stats.gram_dev = max |X^T X - I| of the input (else -1) */
} oracle_opts;

typedef struct {
  double rel_resid;    /* ||A X - X D||_F / ||A - shift I||_inf for this sweep's (post-flip) input */
  double corr_norm;    /* ||E_L||_F */
  double min_gap;      /* min_{i != j} |d_j - d_i| */
  int32_t delta_hits;  /* number of ordered pairs (i,j), i != j, that took the beta branch */
  int32_t flipped;     /* any sigma_j = -1 */
  double gram_dev;     /* max_ij |(X^T X - I)_ij| of the sweep's input (NEXT-4 reorthogonalisation policy) */
} oracle_stats;

/* Optional dumps of the sweep's intermediates (each may be NULL):
 *  [0] W (n x k, post-flip)   [1] Y (n x k)   [2] T (k x k)   [3] sigma (k)
 *  [4] dtilde (k)            [5] alpha (k)    [6] V (n x k)   [7] E (n x k)
 *  [8] Xtilde (n x k, before normalisation)   [9] U (k x k) */
enum { DBG_W = 0, DBG_Y, DBG_T, DBG_SIGMA, DBG_D, DBG_ALPHA, DBG_V, DBG_E, DBG_XT, DBG_U, DBG_N };

static int sweep(const op_t* op, int32_t k, double* X, double normA, const oracle_opts* o,
                 oracle_stats* st, double** dbg) {
  const int64_t n = op->n;
  if (k < 1 || (int64_t)k >= n) return OR_E_INVALID;
  const double u = ldexp(1.0, -53);
  const double delta = o->delta_c * normA * u;
  const size_t nk = (size_t)n * (size_t)k, kk = (size_t)k * (size_t)k;
  double* W = (double*)malloc(sizeof(double) * nk);   /* W -> R -> V -> E in place */
  double* Y = (double*)malloc(sizeof(double) * nk);
  double* T = (double*)malloc(sizeof(double) * kk);
  double* U = (double*)malloc(sizeof(double) * kk);
  double* Z = (double*)malloc(sizeof(double) * kk);
  double* P = (double*)malloc(sizeof(double) * kk);
  double* sig = (double*)malloc(sizeof(double) * (size_t)k);
  double* alpha = (double*)malloc(sizeof(double) * (size_t)k);
  double* d = (double*)malloc(sizeof(double) * (size_t)k);
  double* nrm = (double*)malloc(sizeof(double) * (size_t)k);
  int status = OR_OK;
  double* X0 = (st && o->want_gram) ? (double*)malloc(sizeof(double) * nk) : NULL;
  if (!W || !Y || !T || !U || !Z || !P || !sig || !alpha || !d || !nrm || (st && o->want_gram && !X0)) {
    status = OR_E_NOMEM; goto done;
  }
  if (X0) memcpy(X0, X, sizeof(double) * nk);

  /* line 1: W = A X  (with the Sec. 5.1 shift) */
  op_apply(op, k, X, W);

  /* line 2: Y, T via Alg. 3 (reading: always Alg. 3; Alg. 1 == Alg. 3 after the flip) */
  memcpy(Y, X, sizeof(double) * nk);
  status = oracle_modified_lu(n, k, Y, sig);
  if (status != OR_OK) goto done;
  for (int32_t i = 0; i < k; ++i)
    for (int32_t j = 0; j < k; ++j) U[IDX(i, j, k)] = (j >= i) ? Y[IDX(i, j, k)] : 0.0;
  #pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i)
    for (int32_t j = 0; j < k; ++j)
      if (i <= j) Y[IDX(i, j, k)] = (i == j) ? 1.0 : 0.0;   /* unit lower trapezoidal */
  {
    double* B = Z;  /* scratch: B = -U Sigma */
    for (int32_t i = 0; i < k; ++i)
      for (int32_t j = 0; j < k; ++j) B[IDX(i, j, k)] = -(U[IDX(i, j, k)] * sig[j]);
    solve_right_unit_lower_transpose(k, Y, B, T);
  }
  /* one-time sign transformation X <- X Sigma, and W <- W Sigma
   * so that W = A X still holds (reading R2) */
  int32_t flipped = 0;
  for (int32_t j = 0; j < k; ++j) flipped |= (sig[j] < 0.0);
  if (flipped) {
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i)
      for (int32_t j = 0; j < k; ++j) { X[IDX(i, j, k)] *= sig[j]; W[IDX(i, j, k)] *= sig[j]; }
  }
  if (dbg && dbg[DBG_W]) memcpy(dbg[DBG_W], W, sizeof(double) * nk);

  /* lines 3-4: alpha_j = x_j^T x_j;  d_j = x_j^T w_j / alpha_j   (eq. Rayleigh) */
  #pragma omp parallel for schedule(static)
  for (int32_t j = 0; j < k; ++j) {
    nsum sa = {0, 0}, sg = {0, 0};
    for (int64_t i = 0; i < n; ++i) {
      const double x = X[IDX(i, j, k)];
      nsum_add(&sa, x * x);
      nsum_add(&sg, x * W[IDX(i, j, k)]);
    }
    alpha[j] = nsum_val(&sa);
    d[j] = nsum_val(&sg) / alpha[j];
  }
  for (int32_t j = 0; j < k; ++j) {
    if (!isfinite(alpha[j]) || !isfinite(d[j])) { status = OR_DIVERGED; goto done; }
    if (!(alpha[j] > 0.0)) { status = OR_E_INVALID; goto done; }
    if (fabs(d[j]) <= delta) { status = OR_E_NEAR_ZERO_RQ; goto done; }
  }

  /* line 5: V = H^T (W - X D)  with  H^T B = B - Y (T^T (Y^T B)) */
  #pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i)
    for (int32_t j = 0; j < k; ++j) W[IDX(i, j, k)] = fma(-X[IDX(i, j, k)], d[j], W[IDX(i, j, k)]);  /* R */
  double rr;
  {
    nsum s = {0, 0};
    for (size_t t = 0; t < nk; ++t) nsum_add(&s, W[t] * W[t]);
    rr = nsum_val(&s);
  }
  yt_b(n, k, Y, k, W, Z);                                   /* Z = Y^T R */
  for (int32_t a = 0; a < k; ++a)                           /* P = T^T Z */
    for (int32_t c = 0; c < k; ++c) {
      double s = 0.0;
      for (int32_t l = 0; l < k; ++l) s += T[IDX(l, a, k)] * Z[IDX(l, c, k)];
      P[IDX(a, c, k)] = s;
    }
  #pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i)                           /* V = R - Y P */
    for (int32_t c = 0; c < k; ++c) {
      double s = 0.0;
      for (int32_t l = 0; l < k; ++l) s += Y[IDX(i, l, k)] * P[IDX(l, c, k)];
      W[IDX(i, c, k)] = W[IDX(i, c, k)] - s;
    }
  if (dbg && dbg[DBG_V]) memcpy(dbg[DBG_V], W, sizeof(double) * nk);

  /* line 6: E_L entries (eqs. Ediag, Eoffdiag; delta/beta PAPER.md:443-460) */
  int32_t hits = 0;
  double min_gap = INFINITY;
  for (int32_t i = 0; i < k; ++i)
    for (int32_t j = 0; j < k; ++j) {
      if (o->top_zero) {   /* after Rayleigh-Ritz: e_ij = 0 for i, j <= k */
        if (i != j && fabs(d[j] - d[i]) < min_gap) min_gap = fabs(d[j] - d[i]);
        W[IDX(i, j, k)] = 0.0;
        continue;
      }
      if (i == j) { W[IDX(i, j, k)] = (1.0 - alpha[i]) / 2.0; continue; }
      const double gap = d[j] - d[i];
      if (fabs(gap) < min_gap) min_gap = fabs(gap);
      if (fabs(gap) <= delta) {
        ++hits;
        double beta = 0.0;
        if (!o->beta_zero) {   /* beta_ij = -x_i^T x_j / 2   -- parity unpinned branch */
          nsum s = {0, 0};
          for (int64_t l = 0; l < n; ++l) nsum_add(&s, X[IDX(l, i, k)] * X[IDX(l, j, k)]);
          beta = -nsum_val(&s) / 2.0;
        }
        W[IDX(i, j, k)] = beta;
      } else {
        W[IDX(i, j, k)] = W[IDX(i, j, k)] / gap;
      }
    }
  #pragma omp parallel for schedule(static)
  for (int64_t i = k; i < n; ++i)
    for (int32_t j = 0; j < k; ++j) W[IDX(i, j, k)] = W[IDX(i, j, k)] / d[j];
  if (dbg && dbg[DBG_E]) memcpy(dbg[DBG_E], W, sizeof(double) * nk);

  /* line 7: X~ = X + H E  with  H E = E - Y (T (Y^T E)) */
  double en;
  {
    const int32_t kj = (o->kjudge > 0 && o->kjudge < k) ? o->kjudge : k;
    nsum s = {0, 0};
    for (size_t t = 0; t < nk; ++t)
      if ((int32_t)(t % (size_t)k) < kj) nsum_add(&s, W[t] * W[t]);
    en = nsum_val(&s);
  }
  yt_b(n, k, Y, k, W, Z);                                   /* Qm = Y^T E */
  for (int32_t a = 0; a < k; ++a)                           /* B = T Qm  (into P) */
    for (int32_t c = 0; c < k; ++c) {
      double s = 0.0;
      for (int32_t l = 0; l < k; ++l) s += T[IDX(a, l, k)] * Z[IDX(l, c, k)];
      P[IDX(a, c, k)] = s;
    }
  #pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i)
    for (int32_t c = 0; c < k; ++c) {
      double s = 0.0;
      for (int32_t l = 0; l < k; ++l) s += Y[IDX(i, l, k)] * P[IDX(l, c, k)];
      X[IDX(i, c, k)] = X[IDX(i, c, k)] + (W[IDX(i, c, k)] - s);
    }
  if (dbg && dbg[DBG_XT]) memcpy(dbg[DBG_XT], X, sizeof(double) * nk);

  /* normalise columns (reading R7) */
  if (o->normalize) {
    #pragma omp parallel for schedule(static)
    for (int32_t j = 0; j < k; ++j) {
      nsum s = {0, 0};
      for (int64_t i = 0; i < n; ++i) nsum_add(&s, X[IDX(i, j, k)] * X[IDX(i, j, k)]);
      nrm[j] = sqrt(nsum_val(&s));
    }
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i)
      for (int32_t j = 0; j < k; ++j) X[IDX(i, j, k)] = X[IDX(i, j, k)] / nrm[j];
  }

  if (st) {
    double gd = -1.0;  /* Gram deviation of the (post-flip) input; |entries| are flip-invariant */
    if (X0) {
      gd = 0.0;
      #pragma omp parallel for schedule(static) reduction(max : gd)
      for (int32_t a = 0; a < k; ++a)
        for (int32_t b = 0; b < k; ++b) {
          nsum g = {0, 0};
          for (int64_t i = 0; i < n; ++i) nsum_add(&g, X0[IDX(i, a, k)] * X0[IDX(i, b, k)]);
          const double dv = fabs(nsum_val(&g) - (a == b ? 1.0 : 0.0));
          if (dv > gd) gd = dv;
        }
    }
    st->gram_dev = gd;
    st->rel_resid = sqrt(rr) / normA;
    st->corr_norm = sqrt(en);
    st->min_gap = (k > 1) ? min_gap : 0.0;
    st->delta_hits = hits;
    st->flipped = flipped;
  }
  if (dbg) {
    if (dbg[DBG_Y]) memcpy(dbg[DBG_Y], Y, sizeof(double) * nk);
    if (dbg[DBG_T]) memcpy(dbg[DBG_T], T, sizeof(double) * kk);
    if (dbg[DBG_U]) memcpy(dbg[DBG_U], U, sizeof(double) * kk);
    if (dbg[DBG_SIGMA]) memcpy(dbg[DBG_SIGMA], sig, sizeof(double) * (size_t)k);
    if (dbg[DBG_D]) memcpy(dbg[DBG_D], d, sizeof(double) * (size_t)k);
    if (dbg[DBG_ALPHA]) memcpy(dbg[DBG_ALPHA], alpha, sizeof(double) * (size_t)k);
  }
  for (size_t t = 0; t < nk; ++t)
    if (!isfinite(X[t])) { status = OR_DIVERGED; break; }
done:
  free(W); free(Y); free(T); free(U); free(Z); free(P); free(sig); free(alpha); free(d); free(nrm); free(X0);
  return status;
}

static void fill_opts(oracle_opts* o, double delta_c, int32_t beta_zero, int32_t normalize) {
  o->delta_c = delta_c; o->beta_zero = beta_zero; o->normalize = normalize; o->top_zero = 0; o->kjudge = 0; o->want_gram = 0;
}

int oracle_sweep_dense(int64_t n, int32_t k, const double* A, int64_t lda, double shift,
                       double* X, double delta_c, int32_t beta_zero, int32_t normalize,
                       oracle_stats* st, double** dbg) {
  op_t op = {0, n, A, lda, NULL, NULL, NULL, shift};
  oracle_opts o; fill_opts(&o, delta_c, beta_zero, normalize);
  return sweep(&op, k, X, op_norm_inf(&op), &o, st, dbg);
}

int oracle_sweep_csr(int64_t n, int32_t k, const int32_t* rp, const int32_t* ci, const double* v,
                     double shift, double* X, double delta_c, int32_t beta_zero, int32_t normalize,
                     oracle_stats* st, double** dbg) {
  op_t op = {1, n, NULL, 0, rp, ci, v, shift};
  oracle_opts o; fill_opts(&o, delta_c, beta_zero, normalize);
  return sweep(&op, k, X, op_norm_inf(&op), &o, st, dbg);
}

/* one sweep after Rayleigh-Ritz (top block of E_L zero, beta = 0) */
int oracle_sweep_tz_dense(int64_t n, int32_t k, const double* A, int64_t lda, double shift, double* X,
                          double delta_c, oracle_stats* st, double** dbg) {
  op_t op = {0, n, A, lda, NULL, NULL, NULL, shift};
  oracle_opts o; fill_opts(&o, delta_c, 1, 1); o.top_zero = 1;
  return sweep(&op, k, X, op_norm_inf(&op), &o, st, dbg);
}
int oracle_sweep_tz_csr(int64_t n, int32_t k, const int32_t* rp, const int32_t* ci, const double* v, double shift,
                        double* X, double delta_c, oracle_stats* st, double** dbg) {
  op_t op = {1, n, NULL, 0, rp, ci, v, shift};
  oracle_opts o; fill_opts(&o, delta_c, 1, 1); o.top_zero = 1;
  return sweep(&op, k, X, op_norm_inf(&op), &o, st, dbg);
}

/* =========================================================================
 * The refinement loop (eq. update-X iterated) with the
 * correction-size stopping criterion ||E_L||_F <= tol.
 * Divergence: a non-finite value, or ||E_L||_F growing >= guard_factor within
 * guard_window sweeps ("grows rapidly ... terminate").
 * history (nullable): iters x 2 doubles {rel_resid, corr_norm} per sweep.
 * ========================================================================= */
static int run(const op_t* op, int32_t k, double* X, int32_t iters, double tol, double delta_c,
               int32_t beta_zero, int32_t guard_window, double guard_factor,
               int32_t* iters_done, double* history) {
  oracle_opts o; fill_opts(&o, delta_c, beta_zero, 1);
  const double normA = op_norm_inf(op);
  double* hist_c = (double*)malloc(sizeof(double) * (size_t)(iters > 0 ? iters : 1));
  int status = OR_MAXITER;
  int32_t t = 0;
  for (; t < iters; ++t) {
    oracle_stats st;
    int s = sweep(op, k, X, normA, &o, &st, NULL);
    if (s != OR_OK) { status = s; ++t; break; }
    if (history) { history[2 * t] = st.rel_resid; history[2 * t + 1] = st.corr_norm; }
    hist_c[t] = st.corr_norm;
    if (!isfinite(st.corr_norm)) { status = OR_DIVERGED; ++t; break; }
    if (st.corr_norm <= tol) { status = OR_OK; ++t; break; }
    if (guard_window > 0 && t >= guard_window && st.corr_norm >= guard_factor * hist_c[t - guard_window]) {
      status = OR_DIVERGED; ++t; break;
    }
  }
  if (iters_done) *iters_done = t;
  free(hist_c);
  return status;
}

int oracle_run_dense(int64_t n, int32_t k, const double* A, int64_t lda, double shift, double* X,
                     int32_t iters, double tol, double delta_c, int32_t beta_zero,
                     int32_t guard_window, double guard_factor, int32_t* iters_done, double* history) {
  op_t op = {0, n, A, lda, NULL, NULL, NULL, shift};
  return run(&op, k, X, iters, tol, delta_c, beta_zero, guard_window, guard_factor, iters_done, history);
}
int oracle_run_csr(int64_t n, int32_t k, const int32_t* rp, const int32_t* ci, const double* v,
                   double shift, double* X, int32_t iters, double tol, double delta_c, int32_t beta_zero,
                   int32_t guard_window, double guard_factor, int32_t* iters_done, double* history) {
  op_t op = {1, n, NULL, 0, rp, ci, v, shift};
  return run(&op, k, X, iters, tol, delta_c, beta_zero, guard_window, guard_factor, iters_done, history);
}

/* =========================================================================
 * Rayleigh-Ritz preprocessing for clustered targets (Sec. 3.4):
 *   solve (X^T A X) S = (X^T X) S D~  and set  X <- Z = X S,  so Z^T Z = I and
 *   Z^T A Z = D~; the refinement that follows uses beta = 0
 *   (PAPER.md:460).  The paper does not say how the k x k pencil is solved; the
 *   readings:
 *     RR1  M = X^T (A - shift I) X is symmetrised, M <- (M + M^T)/2.
 *     RR2  the pencil is reduced with the Cholesky factor G = X^T X = L L^T to the
 *          symmetric C = L^{-1} M L^{-T}, whose eigen-decomposition C = Q diag(d) Q^T
 *          is taken by cyclic Jacobi rotations (row-cyclic order, until the
 *          off-diagonal Frobenius mass <= (u ||C||_F)^2, at most 60 sweeps); S = L^{-T} Q.
 *     RR3  Ritz pairs are ordered by descending Ritz value; each column of Q is signed
 *          so that its entry of largest magnitude (first on ties) is positive.
 *   G and M are Neumaier-compensated length-n sums; k x k arithmetic is plain FP64.
 * Returns OR_E_INVALID if G is numerically singular: a Cholesky pivot <= 4 k u G_jj
 * (X rank deficient; reading RR2).
 * ========================================================================= */
static int jacobi_eig(int32_t k, double* C, double* Q, double* d) {
  for (int32_t i = 0; i < k; ++i)
    for (int32_t j = 0; j < k; ++j) Q[IDX(i, j, k)] = (i == j) ? 1.0 : 0.0;
  const double u = ldexp(1.0, -53);
  double fro = 0.0;
  for (int64_t t = 0; t < (int64_t)k * k; ++t) fro += C[t] * C[t];
  for (int sweep_ = 0; sweep_ < 60; ++sweep_) {
    double off = 0.0;
    for (int32_t i = 0; i < k; ++i)
      for (int32_t j = 0; j < k; ++j)
        if (i != j) off += C[IDX(i, j, k)] * C[IDX(i, j, k)];
    if (off <= u * u * fro) break;
    for (int32_t p = 0; p < k - 1; ++p)
      for (int32_t q = p + 1; q < k; ++q) {
        const double apq = C[IDX(p, q, k)];
        if (apq == 0.0) continue;
        const double theta = (C[IDX(q, q, k)] - C[IDX(p, p, k)]) / (2.0 * apq);
        const double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        const double c = 1.0 / sqrt(t * t + 1.0), sn = t * c;
        for (int32_t r = 0; r < k; ++r) {            /* C <- C J (columns p, q) */
          const double cp = C[IDX(r, p, k)], cq = C[IDX(r, q, k)];
          C[IDX(r, p, k)] = c * cp - sn * cq;
          C[IDX(r, q, k)] = sn * cp + c * cq;
        }
        for (int32_t r = 0; r < k; ++r) {            /* C <- J^T C (rows p, q) */
          const double cp = C[IDX(p, r, k)], cq = C[IDX(q, r, k)];
          C[IDX(p, r, k)] = c * cp - sn * cq;
          C[IDX(q, r, k)] = sn * cp + c * cq;
        }
        for (int32_t r = 0; r < k; ++r) {            /* Q <- Q J */
          const double qp = Q[IDX(r, p, k)], qq = Q[IDX(r, q, k)];
          Q[IDX(r, p, k)] = c * qp - sn * qq;
          Q[IDX(r, q, k)] = sn * qp + c * qq;
        }
      }
  }
  for (int32_t j = 0; j < k; ++j) d[j] = C[IDX(j, j, k)];
  return OR_OK;
}

static int rayleigh_ritz(const op_t* op, int32_t k, double* X, double* ritz) {
  const int64_t n = op->n;
  if (k < 1 || (int64_t)k >= n) return OR_E_INVALID;
  const size_t nk = (size_t)n * (size_t)k, kk = (size_t)k * (size_t)k;
  double* W = (double*)malloc(sizeof(double) * nk);
  double* Z = (double*)malloc(sizeof(double) * nk);
  double* G = (double*)malloc(sizeof(double) * kk);
  double* M = (double*)malloc(sizeof(double) * kk);
  double* Cm = (double*)malloc(sizeof(double) * kk);
  double* Q = (double*)malloc(sizeof(double) * kk);
  double* S = (double*)malloc(sizeof(double) * kk);
  double* d = (double*)malloc(sizeof(double) * (size_t)k);
  int32_t* ord = (int32_t*)malloc(sizeof(int32_t) * (size_t)k);
  int status = OR_OK;
  if (!W || !Z || !G || !M || !Cm || !Q || !S || !d || !ord) { status = OR_E_NOMEM; goto done; }
  op_apply(op, k, X, W);                                   /* W = (A - shift I) X */
  #pragma omp parallel for schedule(static)
  for (int32_t a = 0; a < k; ++a)                          /* G = X^T X, M = X^T W */
    for (int32_t b = 0; b < k; ++b) {
      nsum sg = {0, 0}, sm = {0, 0};
      for (int64_t i = 0; i < n; ++i) {
        nsum_add(&sg, X[IDX(i, a, k)] * X[IDX(i, b, k)]);
        nsum_add(&sm, X[IDX(i, a, k)] * W[IDX(i, b, k)]);
      }
      G[IDX(a, b, k)] = nsum_val(&sg);
      M[IDX(a, b, k)] = nsum_val(&sm);
    }
  for (int32_t a = 0; a < k; ++a)                          /* RR1: symmetrise M */
    for (int32_t b = a + 1; b < k; ++b) {
      const double m = (M[IDX(a, b, k)] + M[IDX(b, a, k)]) / 2.0;
      M[IDX(a, b, k)] = m; M[IDX(b, a, k)] = m;
    }
  for (int32_t j = 0; j < k; ++j) {                        /* RR2: G = L L^T (L in G's lower part) */
    double s = G[IDX(j, j, k)];
    const double g0 = s;
    for (int32_t l = 0; l < j; ++l) s -= G[IDX(j, l, k)] * G[IDX(j, l, k)];
    /* numerically singular (X rank deficient): pivot <= 4 k u G_jj */
    if (!(s > 4.0 * k * ldexp(1.0, -53) * g0)) { status = OR_E_INVALID; goto done; }
    const double ljj = sqrt(s);
    G[IDX(j, j, k)] = ljj;
    for (int32_t i = j + 1; i < k; ++i) {
      double t = G[IDX(i, j, k)];
      for (int32_t l = 0; l < j; ++l) t -= G[IDX(i, l, k)] * G[IDX(j, l, k)];
      G[IDX(i, j, k)] = t / ljj;
    }
  }
  /* C = L^{-1} M L^{-T}: B = L^{-1} M (forward substitution per column), C = L^{-1} B^T */
  for (int32_t c = 0; c < k; ++c)
    for (int32_t i = 0; i < k; ++i) {
      double t = M[IDX(i, c, k)];
      for (int32_t l = 0; l < i; ++l) t -= G[IDX(i, l, k)] * Cm[IDX(l, c, k)];
      Cm[IDX(i, c, k)] = t / G[IDX(i, i, k)];
    }
  for (int32_t c = 0; c < k; ++c)                          /* S <- (L^{-1} M)^T, scratch */
    for (int32_t i = 0; i < k; ++i) S[IDX(i, c, k)] = Cm[IDX(c, i, k)];
  for (int32_t c = 0; c < k; ++c)
    for (int32_t i = 0; i < k; ++i) {
      double t = S[IDX(i, c, k)];
      for (int32_t l = 0; l < i; ++l) t -= G[IDX(i, l, k)] * Cm[IDX(l, c, k)];
      Cm[IDX(i, c, k)] = t / G[IDX(i, i, k)];
    }
  for (int32_t a = 0; a < k; ++a)                          /* symmetrise C */
    for (int32_t b = a + 1; b < k; ++b) {
      const double m = (Cm[IDX(a, b, k)] + Cm[IDX(b, a, k)]) / 2.0;
      Cm[IDX(a, b, k)] = m; Cm[IDX(b, a, k)] = m;
    }
  jacobi_eig(k, Cm, Q, d);
  for (int32_t j = 0; j < k; ++j) ord[j] = j;              /* RR3: descending Ritz values */
  for (int32_t a = 1; a < k; ++a) {                        /* insertion sort, stable */
    const int32_t v = ord[a];
    int32_t b = a - 1;
    while (b >= 0 && d[ord[b]] < d[v]) { ord[b + 1] = ord[b]; --b; }
    ord[b + 1] = v;
  }
  for (int32_t j = 0; j < k; ++j) {                        /* permuted, signed Q into Cm */
    const int32_t o = ord[j];
    int32_t im = 0;
    for (int32_t i = 1; i < k; ++i)
      if (fabs(Q[IDX(i, o, k)]) > fabs(Q[IDX(im, o, k)])) im = i;
    const double sg = (Q[IDX(im, o, k)] < 0.0) ? -1.0 : 1.0;
    for (int32_t i = 0; i < k; ++i) Cm[IDX(i, j, k)] = sg * Q[IDX(i, o, k)];
    ritz[j] = d[o];
  }
  for (int32_t c = 0; c < k; ++c)                          /* S = L^{-T} Q (back substitution) */
    for (int32_t i = k - 1; i >= 0; --i) {
      double t = Cm[IDX(i, c, k)];
      for (int32_t l = i + 1; l < k; ++l) t -= G[IDX(l, i, k)] * S[IDX(l, c, k)];
      S[IDX(i, c, k)] = t / G[IDX(i, i, k)];
    }
  #pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i)                          /* Z = X S */
    for (int32_t c = 0; c < k; ++c) {
      double t = 0.0;
      for (int32_t l = 0; l < k; ++l) t += X[IDX(i, l, k)] * S[IDX(l, c, k)];
      Z[IDX(i, c, k)] = t;
    }
  memcpy(X, Z, sizeof(double) * nk);
  for (size_t t = 0; t < nk; ++t)
    if (!isfinite(X[t])) { status = OR_DIVERGED; break; }
done:
  free(W); free(Z); free(G); free(M); free(Cm); free(Q); free(S); free(d); free(ord);
  return status;
}

int oracle_rr_dense(int64_t n, int32_t k, const double* A, int64_t lda, double shift, double* X, double* ritz) {
  op_t op = {0, n, A, lda, NULL, NULL, NULL, shift};
  return rayleigh_ritz(&op, k, X, ritz);
}
int oracle_rr_csr(int64_t n, int32_t k, const int32_t* rp, const int32_t* ci, const double* v, double shift,
                  double* X, double* ritz) {
  op_t op = {1, n, NULL, 0, rp, ci, v, shift};
  return rayleigh_ritz(&op, k, X, ritz);
}
/* k x k symmetric eigen-decomposition alone (tests): C (in, destroyed) -> Q, d (unsorted) */
int oracle_jacobi_eig(int32_t k, double* C, double* Q, double* d) { return jacobi_eig(k, C, Q, d); }

/* Extended entry points: square = 1 -> operator A^2 - shift I (Sec. 5.2);
 * kjudge > 0 -> refine all k columns, judge (corr_norm, stopping) on the leading kjudge (K > k,
 * PAPER.md:941-942, 958-967).  is_csr selects the dense (A, lda) or CSR (rp, ci, v) operand. */
int oracle_sweep_ex(int is_csr, int64_t n, int32_t k, const double* A, int64_t lda, const int32_t* rp,
                    const int32_t* ci, const double* v, double shift, int32_t square, double* X, double delta_c,
                    int32_t beta_zero, int32_t kjudge, int32_t want_gram, oracle_stats* st, double** dbg) {
  op_t op = {is_csr, n, A, lda, rp, ci, v, shift, square};
  oracle_opts o; fill_opts(&o, delta_c, beta_zero, 1); o.kjudge = kjudge; o.want_gram = want_gram;
  return sweep(&op, k, X, op_norm_inf(&op), &o, st, dbg);
}
int oracle_run_ex(int is_csr, int64_t n, int32_t k, const double* A, int64_t lda, const int32_t* rp,
                  const int32_t* ci, const double* v, double shift, int32_t square, double* X, int32_t iters,
                  double tol, double delta_c, int32_t beta_zero, int32_t kjudge, int32_t* iters_done,
                  double* history) {
  op_t op = {is_csr, n, A, lda, rp, ci, v, shift, square};
  oracle_opts o; fill_opts(&o, delta_c, beta_zero, 1); o.kjudge = kjudge;
  const double normA = op_norm_inf(&op);
  int status = OR_MAXITER;
  int32_t t = 0;
  for (; t < iters; ++t) {
    oracle_stats s_;
    const int s = sweep(&op, k, X, normA, &o, &s_, NULL);
    if (s != OR_OK) { status = s; ++t; break; }
    if (history) { history[2 * t] = s_.rel_resid; history[2 * t + 1] = s_.corr_norm; }
    if (!isfinite(s_.corr_norm)) { status = OR_DIVERGED; ++t; break; }
    if (s_.corr_norm <= tol) { status = OR_OK; ++t; break; }
  }
  if (iters_done) *iters_done = t;
  return status;
}
int oracle_apply_ex(int is_csr, int64_t n, int32_t k, const double* A, int64_t lda, const int32_t* rp,
                    const int32_t* ci, const double* v, double shift, int32_t square, const double* X, double* W) {
  op_t op = {is_csr, n, A, lda, rp, ci, v, shift, square};
  op_apply(&op, k, X, W);
  return OR_OK;
}
double oracle_norm_ex(int is_csr, int64_t n, const double* A, int64_t lda, const int32_t* rp, const int32_t* ci,
                      const double* v, double shift, int32_t square) {
  op_t op = {is_csr, n, A, lda, rp, ci, v, shift, square};
  return op_norm_inf(&op);
}

/* =========================================================================
 * Reorthogonalisation ("optionally reorthogonalize"): Cholesky QR,
 * X <- X L^{-T} with X^T X = L L^T (Neumaier Gram, plain k x k arithmetic), so the columns become
 * orthonormal and span(X) is kept.  gram_dev (nullable): max |X^T X - I| before.  OR_E_INVALID if a
 * pivot <= 4 k u G_jj (X rank deficient).
 * ========================================================================= */
int oracle_reorthogonalize(int64_t n, int32_t k, double* X, double* gram_dev) {
  const size_t kk = (size_t)k * (size_t)k;
  double* G = (double*)malloc(sizeof(double) * kk);
  double* row = (double*)malloc(sizeof(double) * (size_t)k);
  if (!G || !row) { free(G); free(row); return OR_E_NOMEM; }
  double gd = 0.0;
  for (int32_t a = 0; a < k; ++a)
    for (int32_t b = 0; b < k; ++b) {
      nsum g = {0, 0};
      for (int64_t i = 0; i < n; ++i) nsum_add(&g, X[IDX(i, a, k)] * X[IDX(i, b, k)]);
      G[IDX(a, b, k)] = nsum_val(&g);
      const double dv = fabs(G[IDX(a, b, k)] - (a == b ? 1.0 : 0.0));
      if (dv > gd) gd = dv;
    }
  if (gram_dev) *gram_dev = gd;
  for (int32_t j = 0; j < k; ++j) {                 /* G = L L^T (lower) */
    double sj = G[IDX(j, j, k)];
    const double g0 = sj;
    for (int32_t l = 0; l < j; ++l) sj -= G[IDX(j, l, k)] * G[IDX(j, l, k)];
    if (!(sj > 4.0 * k * ldexp(1.0, -53) * g0)) { free(G); free(row); return OR_E_INVALID; }
    const double ljj = sqrt(sj);
    G[IDX(j, j, k)] = ljj;
    for (int32_t i = j + 1; i < k; ++i) {
      double t = G[IDX(i, j, k)];
      for (int32_t l = 0; l < j; ++l) t -= G[IDX(i, l, k)] * G[IDX(j, l, k)];
      G[IDX(i, j, k)] = t / ljj;
    }
  }
  for (int64_t i = 0; i < n; ++i) {                 /* row x_i <- x_i L^{-T}: solve z L^T = x_i */
    for (int32_t j = 0; j < k; ++j) {
      double t = X[IDX(i, j, k)];
      for (int32_t l = 0; l < j; ++l) t -= row[l] * G[IDX(j, l, k)];
      row[j] = t / G[IDX(j, j, k)];
    }
    for (int32_t j = 0; j < k; ++j) X[IDX(i, j, k)] = row[j];
  }
  free(G); free(row);
  return OR_OK;
}

int oracle_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
