// kxk.cuh -- the serial k x k stages of a sweep, each one CTA (k <= 128).
//
// kxk_prep   (S2 + S3): fixed-order reduction of the alpha/g double-double partials
//            -> alpha_j, d_j = g_j / alpha_j (eq. Rayleigh, Alg. 4
//            lines 3-4); modified LU of the top k x k block X^_1 (Alg. 2, PAPER.md:
//            271-284, sign(0) = +1) -> Sigma, U, Y_1 = L; T = -U Sigma Y_1^{-T}
//            (Alg. 3).  Rows l > k of Alg. 2 only read U's rows, so
//            Y_2 = X^_2 U^{-1} (the tall-skinny triangular apply) is never formed on
//            the hot path: it is applied through k x k algebra.
// kxk_finish (S4-S6 top block + all k x k algebra): with the one-time flip
//            X' = X^ Sigma, W' = W Sigma, U' = U Sigma (reading R2):
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
// norm_reduce: fixed-order column norms of X~ -> 1/||x~_j||.
#pragma once
#include "common.cuh"

namespace rf {

// ---------------------------------------------------------------- kxk_prep
__global__ void __launch_bounds__(1024) kxk_prep_kernel(Ws ws, const double* __restrict__ Xtop) {
  extern __shared__ __align__(16) double Q[];     // k x k, in-place modified LU
  __shared__ dd pa[1024], pg[1024];
  __shared__ int s_bad;
  if (*ws.status != ST_OK) return;
  const int k = ws.k, tid = threadIdx.x, nt = blockDim.x;

  // 1. alpha_j, g_j: P parts per column, each part a contiguous slot range, combined in order
  const int P = nt / k;
  const int j = tid % k, p = tid / k;
  dd a = {0.0, 0.0}, g = {0.0, 0.0};
  if (p < P) {
    const int s0 = (int)((int64_t)ws.n_ag * p / P), s1 = (int)((int64_t)ws.n_ag * (p + 1) / P);
    for (int s = s0; s < s1; ++s) {
      const double* slot = ws.ag + ((int64_t)s * k + j) * 4;
      dd_add(a, dd{slot[0], slot[1]});
      dd_add(g, dd{slot[2], slot[3]});
    }
  }
  pa[tid] = a;
  pg[tid] = g;
  for (int e = tid; e < k * k; e += nt) Q[e] = Xtop[e];
  if (tid == 0) s_bad = ST_OK;
  __syncthreads();
  if (tid < k) {
    dd ta = pa[tid], tg = pg[tid];
    for (int q = 1; q < P; ++q) { dd_add(ta, pa[q * k + tid]); dd_add(tg, pg[q * k + tid]); }
    const double al = dd_val(ta), gv = dd_val(tg);
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
  __syncthreads();

  // 2. Alg. 2 on the top block, literal order: sigma_j = -sign(q_jj) (sign(0)=+1),
  //    q_jj -= sigma_j, scale the column below, rank-1 update of the trailing block.
  for (int jj = 0; jj < k; ++jj) {
    const double q = Q[jj * k + jj];
    const double s = (q >= 0.0) ? -1.0 : 1.0;
    const double piv = __dadd_rn(q, -s);
    if (piv == 0.0) {                       // uniform across the block
      if (tid == 0) atomicCAS(&s_bad, ST_OK, ST_E_ZERO_PIVOT);
      break;
    }
    __syncthreads();                         // everyone has read q before it is overwritten
    if (tid == 0) { Q[jj * k + jj] = piv; ws.sigma[jj] = s; }
    for (int l = jj + 1 + tid; l < k; l += nt) Q[l * k + jj] = __ddiv_rn(Q[l * k + jj], piv);
    __syncthreads();
    const int m = k - jj - 1;
    for (int e = tid; e < m * m; e += nt) {
      const int l = jj + 1 + e / m, h = jj + 1 + e % m;
      Q[l * k + h] = __dadd_rn(Q[l * k + h], -__dmul_rn(Q[l * k + jj], Q[jj * k + h]));
    }
    __syncthreads();
  }
  __syncthreads();
  for (int e = tid; e < k * k; e += nt) {
    const int r = e / k, c = e % k;
    ws.U[e] = (c >= r) ? Q[e] : 0.0;
    ws.L[e] = (c < r) ? Q[e] : (c == r ? 1.0 : 0.0);
  }
  __syncthreads();

  // 3. T = -U Sigma L^{-T}: row i, ascending j >= i: t_ij = -u_ij sigma_j - sum_{i<=l<j} t_il L_jl
  if (tid < k) {
    const int i = tid;
    double* Ti = ws.T + i * k;
    for (int c = 0; c < i; ++c) Ti[c] = 0.0;
    for (int c = i; c < k; ++c) {
      double t = -(Q[i * k + c] * ws.sigma[c]);
      for (int l = i; l < c; ++l) t = __dadd_rn(t, -__dmul_rn(Ti[l], Q[c * k + l]));
      Ti[c] = t;
    }
  }
  if (tid == 0 && s_bad != ST_OK) *ws.status = s_bad;
}

// ---------------------------------------------------------------- k x k helpers (block-wide)
// C = op(A) op(B) (+ Cadd), all k x k, row-major ld k.  No aliasing of C with inputs.
__device__ void blk_mm(int k, const double* A, bool ta, const double* B, bool tb, double* C,
                       const double* Cadd = nullptr, double add_sign = 1.0) {
  for (int e = threadIdx.x; e < k * k; e += blockDim.x) {
    const int i = e / k, j = e % k;
    double s = 0.0;
    for (int l = 0; l < k; ++l) {
      const double a = ta ? A[l * k + i] : A[i * k + l];
      const double b = tb ? B[j * k + l] : B[l * k + j];
      s = fma(a, b, s);
    }
    C[e] = Cadd ? fma(add_sign, s, Cadd[e]) : s;
  }
}
// X = Up^{-T} M  (Up upper, so Up^T lower: forward substitution), one thread per column
__device__ void blk_solve_upT(int k, const double* Up, const double* M, double* X) {
  for (int c = threadIdx.x; c < k; c += blockDim.x)
    for (int i = 0; i < k; ++i) {
      double s = M[i * k + c];
      for (int l = 0; l < i; ++l) s = fma(-Up[l * k + i], X[l * k + c], s);
      X[i * k + c] = s / Up[i * k + i];
    }
}
// X = Up^{-1} M (back substitution), one thread per column
__device__ void blk_solve_up(int k, const double* Up, const double* M, double* X) {
  for (int c = threadIdx.x; c < k; c += blockDim.x)
    for (int i = k - 1; i >= 0; --i) {
      double s = M[i * k + c];
      for (int l = i + 1; l < k; ++l) s = fma(-Up[i * k + l], X[l * k + c], s);
      X[i * k + c] = s / Up[i * k + i];
    }
}

// ---------------------------------------------------------------- kxk_finish
// Xtop/Wtop: the top k rows of X^ (in/out) and W (un-flipped), ld k.
__global__ void __launch_bounds__(1024) kxk_finish_kernel(Ws ws, double* __restrict__ Xtop,
                                                          const double* __restrict__ Wtop) {
  if (*ws.status != ST_OK) return;
  __shared__ int s_hits;
  __shared__ double s_red[4][KMAX];
  const int k = ws.k, kk = k * k, tid = threadIdx.x, nt = blockDim.x;
  double* S = ws.scratch;
  double *Xp = S, *R1 = S + kk, *Mp = S + 2 * kk, *Gp = S + 3 * kk, *Up = S + 4 * kk, *Z2 = S + 5 * kk,
         *Z = S + 6 * kk, *P = S + 7 * kk, *V1 = S + 8 * kk, *Pt = S + 9 * kk, *GPt = S + 10 * kk,
         *S2 = S + 11 * kk, *Y2E = S + 12 * kk, *Qm = S + 13 * kk, *B = S + 14 * kk, *UB = S + 15 * kk;
  const double* sig = ws.sigma;
  const double* d = ws.d;
  if (tid == 0) s_hits = 0;
  for (int e = tid; e < kk; e += nt) {
    const int i = e / k, j = e % k;
    const double xp = Xtop[e] * sig[j];
    Xp[e] = xp;
    R1[e] = fma(-xp, d[j], Wtop[e] * sig[j]);
    Mp[e] = sig[i] * ws.M2[e] * sig[j];
    Gp[e] = sig[i] * ws.G2[e] * sig[j];
    Up[e] = ws.U[e] * sig[j];
  }
  __syncthreads();
  blk_solve_upT(k, Up, Mp, Z2);                       // U'^{-T} M'
  __syncthreads();
  blk_mm(k, ws.L, true, R1, false, Z, Z2);            // Z = L^T R_1 + U'^{-T} M'
  __syncthreads();
  blk_mm(k, ws.T, true, Z, false, P);                 // P = T^T Z
  __syncthreads();
  blk_mm(k, ws.L, false, P, false, V1, R1, -1.0);     // V_1 = R_1 - L P
  __syncthreads();
  blk_solve_up(k, Up, P, Pt);                         // P~ = U'^{-1} P
  // E_11 (line 6): beta needs the Gram G = X'^T X' = X'_1^T X'_1 + G'
  for (int e = tid; e < kk; e += nt) {
    const int i = e / k, j = e % k;
    double v;
    if (i == j) {
      v = (1.0 - ws.alpha[i]) / 2.0;
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
    ws.E11[e] = v;
  }
  __syncthreads();
  blk_mm(k, Gp, false, Pt, false, GPt);               // G' P~
  __syncthreads();
  for (int e = tid; e < kk; e += nt) S2[e] = (Mp[e] - GPt[e]) / d[e % k];
  __syncthreads();
  blk_solve_upT(k, Up, S2, Y2E);                      // Y_2^T E_2
  __syncthreads();
  blk_mm(k, ws.L, true, ws.E11, false, Qm, Y2E);      // Qm = L^T E_11 + Y_2^T E_2
  __syncthreads();
  blk_mm(k, ws.T, false, Qm, false, B);               // B = T Qm
  __syncthreads();
  blk_solve_up(k, Up, B, UB);                         // U'^{-1} B
  // X~_1 = X'_1 + (E_11 - L B)
  for (int e = tid; e < kk; e += nt) {
    const int i = e / k, j = e % k;
    double s = 0.0;
    for (int l = 0; l < k; ++l) s = fma(ws.L[i * k + l], B[l * k + j], s);
    Xtop[e] = Xp[e] + (ws.E11[e] - s);
  }
  __syncthreads();
  for (int e = tid; e < kk; e += nt) {
    const int l = e / k, j = e % k;
    ws.Csig[e] = sig[l] * (Pt[e] / d[j] + UB[e]);
  }
  // per-column quantities and statistics
  if (tid < k) {
    const int j = tid;
    double nt2 = 0.0, r1 = 0.0, e1 = 0.0, pm = 0.0, pgp = 0.0;
    for (int i = 0; i < k; ++i) {
      const double x = Xtop[i * k + j];
      nt2 = fma(x, x, nt2);
      r1 = fma(R1[i * k + j], R1[i * k + j], r1);
      e1 = fma(ws.E11[i * k + j], ws.E11[i * k + j], e1);
      pm = fma(Pt[i * k + j], Mp[i * k + j], pm);
      pgp = fma(Pt[i * k + j], GPt[i * k + j], pgp);
    }
    ws.ntop[j] = nt2;
    ws.scal[j] = sig[j] / d[j];
    const double e2 = (ws.rr2[j] - 2.0 * pm + pgp) / (d[j] * d[j]);
    s_red[0][j] = r1 + ws.rr2[j];
    s_red[1][j] = e1 + e2;
    double mg = INFINITY;
    for (int i = 0; i < k; ++i)
      if (i != j) mg = fmin(mg, fabs(d[j] - d[i]));
    s_red[2][j] = mg;
    s_red[3][j] = (sig[j] < 0.0) ? 1.0 : 0.0;
  }
  __syncthreads();
  if (tid == 0) {
    double rr = 0.0, en = 0.0, mg = INFINITY, fl = 0.0;
    for (int j = 0; j < k; ++j) { rr += s_red[0][j]; en += s_red[1][j]; mg = fmin(mg, s_red[2][j]); fl += s_red[3][j]; }
    ws.stats[0] = sqrt(rr) / ws.normA;
    ws.stats[1] = sqrt(fmax(en, 0.0));
    ws.stats[2] = (k > 1) ? mg : 0.0;
    ws.stats[3] = (double)s_hits;
    ws.stats[4] = (fl > 0.0) ? 1.0 : 0.0;
    ws.stats[5] = rr;
  }
}

// ---------------------------------------------------------------- norm_reduce
__global__ void __launch_bounds__(128) norm_reduce_kernel(Ws ws) {
  if (*ws.status != ST_OK) return;
  const int j = threadIdx.x;
  if (j >= ws.k) return;
  double s = ws.ntop[j];
  for (int q = 0; q < ws.n_nslot; ++q) s += ws.nslot[(int64_t)q * ws.kp + j];
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
