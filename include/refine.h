/*
 * refine.h -- C ABI of the B200-native refinement sweep (paper_2602_23778_b200).
 *
 * One refinement sweep of arXiv 2602.23778, Algorithm 4:
 * given k << n approximate eigenvectors X^ of a real symmetric n x n matrix A,
 *   W = A X^                              (line 1; shifted A - shift I, Sec. 5.1)
 *   Y^, T^ from X^ by CompactWY_LU        (line 2; Alg. 2, Alg. 3)
 *   alpha_j = x_j^T x_j, d_j = x_j^T w_j / alpha_j        (lines 3-4, eq. Rayleigh)
 *   V = H^T (W - X^ D)                    (line 5, eq. V-def; H = I - Y T Y^T)
 *   E_L from V, d, alpha, delta, beta     (line 6, eqs. Ediag/Eoffdiag PAPER.md:395-426, 443-460)
 *   X^ <- X^ + H E_L                      (line 7, eq. update-X)
 * followed by column normalisation.  The sign transformation
 * X^ <- X^ Sigma of PAPER.md:304-306 is applied inside every sweep (DESIGN.md
 * reading R2), so column signs of X may flip (reported in stats.flipped).
 *
 * All arithmetic is FP64.  Every entry point is extern "C"
 * and takes only plain pointers and sizes; nothing is thrown across the ABI.
 *
 * Memory:  pointers documented "device" are CUDA device pointers on the
 * context's device; "host" pointers are ordinary (preferably pinned) host
 * memory.  Blocks of size n x k are ROW-MAJOR with leading dimension k
 * (entry (i, j) at [i*k + j]).
 *
 * Streams: `stream` is a cudaStream_t passed as void* (NULL = legacy default
 * stream).  All work is enqueued on it; calls return without a host sync
 * unless documented otherwise.  One context per stream; a context is not
 * re-entrant.
 *
 * Errors: every call returns a refine_status.  CUDA and NCCL errors are sticky
 * on the context (every later call returns the same error).  Device-side
 * conditions (near-zero Rayleigh quotient, zero pivot, non-finite values) are
 * detected on the device and reach the host when stats are requested, on
 * refine_run's checks, or via refine_get_status().  When such a condition is
 * detected the sweep leaves X unmodified.
 */
#ifndef PAPER_2602_23778_REFINE_H
#define PAPER_2602_23778_REFINE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct refine_ctx refine_ctx;   /* opaque; owned by the library */

typedef enum {
  REFINE_OK = 0,               /* refine_run: ||E_L||_F <= tol; otherwise success          */
  REFINE_MAXITER = 1,          /* refine_run: iteration budget exhausted                                  */
  REFINE_DIVERGED = 2,         /* non-finite value, or ||E_L||_F grew >= guard_factor within guard_window
                                  sweeps                                                  */
  REFINE_E_INVALID = -1,       /* bad argument: k < 1, k >= n, lda < n, NULL, CSR out of range, alpha<=0  */
  REFINE_E_NEAR_ZERO_RQ = -2,  /* |d_j| <= delta (PAPER.md:443-446 divides by d_j): shift A (Sec. 5)       */
  REFINE_E_ZERO_PIVOT = -3,    /* modified-LU pivot exactly zero (Alg. 2 line 4; defensive)               */
  REFINE_E_CUDA = -4,          /* CUDA runtime error (sticky)                                             */
  REFINE_E_NCCL = -5,          /* NCCL error (sticky)                                                     */
  REFINE_E_NOMEM = -6,         /* device allocation failed                                                */
  REFINE_E_UNSUPPORTED = -7    /* k above the compiled maximum (128) or another unsupported shape         */
} refine_status;

/* Process group of the row partition (one process per GPU).  world == 1:
 * everything local, nccl_id ignored.  world > 1 with nccl_id != NULL: rank r owns
 * rows [row_begin, row_end) of A and X^ (the ranks' ranges must tile [0, n) in
 * rank order; rank 0 must own rows 0..k-1); nccl_id is the 128-byte
 * ncclUniqueId produced by refine_nccl_id() on rank 0 and broadcast by the
 * caller (e.g. torch.distributed); the caller has selected the rank's device.
 * Per sweep the ranks exchange X (dense: every block to every rank; CSR: only
 * the halo rows the local rows reference) and gather small per-rank partials
 * (2k, 2k^2 + k and k doubles) and one broadcast of k^2 + k + 9 doubles from
 * rank 0; every cross-rank sum is taken in rank order, so the k x k state is
 * bit-identical on all ranks.
 * world > 1 with nccl_id == NULL: LOOPBACK emulation for tests -- one process,
 * one device, the FULL problem is passed (row_begin = 0, row_end = n) and split
 * into `world` row blocks that run the multi-rank code path with device copies
 * in place of NCCL. */
typedef struct {
  int32_t rank;
  int32_t world;
  const void* nccl_id;
} refine_comm;

/* Options (NULL = defaults). */
typedef struct {
  double delta_c;        /* delta = delta_c * ||A - shift I||_inf * 2^-53; default 10 */
  int32_t beta_zero;     /* 0: beta_ij = -x_i^T x_j / 2; 1: beta_ij = 0      */
  int32_t normalize;     /* 1: normalise columns after each update; default 1              */
  int32_t guard_window;  /* refine_run divergence guard window, 0..4 (0 = off; outside -> REFINE_E_INVALID
                            at init); default 3                                                          */
  double guard_factor;   /* refine_run divergence guard growth factor; default 10                         */
  int32_t square;        /* 1: the operator is A^2 - shift I applied as A (A X) (Sec. 5.2, PAPER.md:1218-1243;
                            smallest-|lambda| targets); ||.|| in delta / rel_resid is ||A||_inf^2 + |shift|
                            (reading SQ1).  At world > 1 the rows of T = A X are exchanged between the two
                            products (halo / all-gather, as for X).  Default 0                            */
  int32_t kjudge;        /* > 0: refine all k columns but judge ||E_L||_F (stats, refine_run's stopping
                            test) on the leading kjudge columns (K > k).  Default 0 = all */
  double resid_tol;      /* > 0: refine_run also stops (REFINE_OK) when rel_resid <= resid_tol
                            (PAPER.md:495-499).  Default 0 = off                                            */
  double reorth_tol;     /* > 0: sweeps report gram_dev, and refine_run reorthogonalises (Cholesky QR,
                            refine_reorthogonalize) the output of every sweep whose input had
                            gram_dev > reorth_tol.  world == 1: behind a device gate (no host
                            sync); world > 1: the host reads the gate after each sweep.  Default 0 = off */
  int32_t rr_fallback;   /* 1: when refine_run's divergence guard trips, continue with refine_sweep_rr
                            iterations instead of returning REFINE_DIVERGED        */
  int32_t mixed;         /* NEXT-2 ("matrix-matrix multiplications in the applications
                            of H and H^T may be computed in lower precision while keeping the
                            accumulation and the small k x k computations in double"): 1 = the sweep's
                            tall-skinny products X_2^T [R_2 | X_2] (pass B) and X_2 Csig (pass C) on the
                            bf16 tensor cores (tcgen05) with every FP64 operand split into two bf16
                            terms (three products, relative error ~1e-5 of an O(residual) quantity);
                            R = W - X D, the w scaling, every k x k step and all reductions stay FP64.
                            The sweep still converges to FP64 accuracy, at a per-sweep rate
                            max(gamma, ~1e-5 kappa).  Requires k a multiple of 16, k >= 32 (else
                            REFINE_E_UNSUPPORTED)
                            and a 16-byte aligned X (else the FP64 passes run).  1: pass C (2k^2
                            flop vs 24k bytes per row) uses the tensor cores only for k > 64 where the
                            FP64 pass is compute bound; 2: both passes on tcgen05 at every k.  Rayleigh-Ritz and
                            reorthogonalisation steps always run in FP64 (their products are O(1)). */
  int32_t emul;          /* dense A only: 1 = S1 (W = A X^) with FP64 accuracy on the INT8 tensor cores
                            (Ozaki splitting, ozaki.cuh): A's rows are scaled to their off-diagonal
                            max and cut into 7 balanced base-256 int8 digits (54 bits) ONCE at init
                            (n_loc x n x 7 bytes extra device memory; the diagonal stays FP64), X^'s
                            columns likewise every sweep; the slice products are exact int32 sums on
                            tcgen05.mma kind::i8, combined in FP64.  Error <= 8.2 2^-52 max|A_i.| max|X_.j|
                            per product term: relative to the row and column MAXIMA (rows with a very
                            wide dynamic range should use DMMA).
                            0 (default) = DMMA FP64.  For k == 128 (dense or CSR) it also runs pass C
                            (X_2 Csig, the sweep's O(residual) correction) on kind::i8 with 5 x 7-bit
                            digits per operand, row / column exponents and exact int32 levels: ~2^-35
                            relative to row / column maxima of a correction term -- one-step parity
                            with the FP64 oracle (1e-10) and the FP64 accuracy at convergence kept.
                            Requires (dense, k a multiple of 16, k <= 64) or k == 128 (else
                            REFINE_E_UNSUPPORTED). */
} refine_opts;

/* Per-sweep diagnostics (host struct), for the sweep's input X^ (after the sign flip). */
typedef struct {
  double rel_resid;      /* ||A X^ - X^ D||_F / ||A - shift I||_inf                 */
  double corr_norm;      /* ||E_L||_F                     */
  double min_gap;        /* min_{i != j} |d_j - d_i| over the k Rayleigh quotients                       */
  int32_t delta_hits;    /* ordered pairs (i, j), i != j, that took the beta branch        */
  int32_t flipped;       /* 1 if any sigma_j = -1 this sweep (X^ <- X^ Sigma)           */
  double gram_dev;       /* max |X^T X - I| of the sweep's input when opts.reorth_tol > 0, else -1          */
} refine_sweep_stats;

/* Dense symmetric A (both triangles), FP64, row-major, device pointer.
 * A_rows points at row row_begin of A; rows [row_begin, row_end) are local,
 * each of length n with leading dimension lda >= n.  A is BORROWED: keep it
 * alive and unmodified until refine_destroy.  shift: operator is A - shift*I
 * (PAPER.md:1203).  Allocates every workspace (O(n_loc k + k^2)); computes
 * ||A - shift I||_inf once (one pass over A).  On success *out is a new
 * context; on error *out is NULL. */
refine_status refine_init_dense(refine_ctx** out, int64_t n, int32_t k,
                                const double* A_rows, int64_t lda,
                                int64_t row_begin, int64_t row_end, double shift,
                                const refine_comm* comm, const refine_opts* opts, void* stream);

/* CSR symmetric A (both triangles stored), device pointers: row_ptr has
 * (row_end - row_begin + 1) int32 entries that index col_idx / val directly
 * (absolute offsets; row_ptr[0] may be nonzero, e.g. a row slice of a global
 * CSR), col_idx are GLOBAL int32 column indices sorted ascending within each
 * row, val FP64.  Borrowed like the dense A.  Within a row the
 * product is an fma chain in ascending CSR order (bit-reproducible). */
refine_status refine_init_csr(refine_ctx** out, int64_t n, int32_t k,
                              const int32_t* row_ptr, const int32_t* col_idx, const double* val,
                              int64_t row_begin, int64_t row_end, double shift,
                              const refine_comm* comm, const refine_opts* opts, void* stream);

/* One sweep on X (device, (row_end-row_begin) x k row-major), in place.
 * stats == NULL: fully asynchronous.  stats != NULL: the call synchronises the
 * stream and returns the device status of this sweep. */
refine_status refine_sweep(refine_ctx* c, double* X, refine_sweep_stats* stats);

/* Same sweep with HOST buffers (end-to-end entry point): copies X_host_in
 * (n_loc x k) to the device, runs one sweep, copies the result to X_host_out
 * (may equal X_host_in) and synchronises.  Pinned memory gives full PCIe rate.
 * Dense A, one rank, >= 1 MiB of X: the upload goes in chunks on a copy stream
 * and S1 (the TMA GEMM) consumes each chunk as it lands (per-chunk flags); the
 * result is bit-identical to the device-buffer sweep.  An upload that never
 * completes ends the sweep with REFINE_DIVERGED after 5 s instead of hanging.
 * REFINE_H2D_OVERLAP=0 uploads everything before the sweep. */
refine_status refine_sweep_host(refine_ctx* c, const double* X_host_in, double* X_host_out,
                                refine_sweep_stats* stats);

/* Iterate sweeps on X (device) until ||E_L||_F <= tol (REFINE_OK), iters sweeps
 * (REFINE_MAXITER), divergence (REFINE_DIVERGED) or a device error.  Synchronises.
 * iters_done / last (nullable) report the sweeps executed and the last stats.
 * opts.resid_tol / reorth_tol / rr_fallback add the NEXT-4 policies (see refine_opts);
 * the plain loop runs without host synchronisation (device-side halting). */
refine_status refine_run(refine_ctx* c, double* X, int32_t iters, double tol,
                         int32_t* iters_done, refine_sweep_stats* last);

/* Rayleigh-Ritz preprocessing for clustered targets (Sec. 3.4):
 * solves (X^T A' X) S = (X^T X) S D~ (A' = A - shift I) and replaces X (device,
 * n_loc x k row-major, in place) by Z = X S, so Z^T Z = I and Z^T A' Z = D~
 * (PAPER.md:915-919).  The k x k pencil is reduced by the Cholesky factor of X^T X
 * and solved by parallel Jacobi rotations on one CTA; Ritz pairs are ordered by
 * descending Ritz value, each eigenvector column signed so its largest entry is
 * positive (readings RR1-RR3).  ritz (host, k doubles, nullable) receives
 * D~ (on every rank of a row partition: the values are broadcast with the k x k state).
 * Synchronises.  REFINE_E_INVALID if X^T X is not positive definite (X rank
 * deficient); X is then unchanged. */
refine_status refine_rayleigh_ritz(refine_ctx* c, double* X, double* ritz);

/* Reorthogonalisation ("optionally reorthogonalize"): Cholesky QR,
 * X <- X L^{-T} with X^T X = L L^T (columns orthonormal, span kept).  gram_dev (host,
 * nullable) receives max |X^T X - I| before (every rank).  Synchronises.  REFINE_E_INVALID if X is
 * rank deficient (X unchanged). */
refine_status refine_reorthogonalize(refine_ctx* c, double* X, double* gram_dev);

/* One iteration of the preprocessed refinement: refine_rayleigh_ritz, then one sweep
 * whose E_L top block is set to its exact-arithmetic value 0 (beta = 0,
 * PAPER.md:460).  Stats / ritz as for refine_sweep / refine_rayleigh_ritz.  Synchronises. */
refine_status refine_sweep_rr(refine_ctx* c, double* X, refine_sweep_stats* stats, double* ritz);

/* Status of the last enqueued sweep (synchronises the stream). */
refine_status refine_get_status(refine_ctx* c);

/* Capture the sweep for X as a CUDA graph and replay it on later calls with the
 * same X pointer (enable = 1), or launch kernels directly (enable = 0, default). */
refine_status refine_set_graph(refine_ctx* c, int32_t enable);

/* Number of CUDA kernel launches one sweep enqueues (for the bench's gpu_launches). */
int32_t refine_kernels_per_sweep(const refine_ctx* c);

/* Live per-kernel timing (bench.py's roofline): after refine_profile_begin, every sweep
 * enqueued (without graphs) records a CUDA event at each kernel boundary on the context's
 * stream; refine_profile_end synchronises and writes, for each of the
 * refine_kernels_per_sweep() kernels, the summed milliseconds over the recorded sweeps
 * (ms_sum must hold that many doubles).  refine_kernel_name(i) names kernel i. */
refine_status refine_profile_begin(refine_ctx* c, int32_t max_sweeps);
refine_status refine_profile_end(refine_ctx* c, double* ms_sum, int32_t* nkernels, int32_t* nsweeps);
const char* refine_kernel_name(const refine_ctx* c, int32_t i);

void refine_destroy(refine_ctx* c);
const char* refine_status_string(refine_status s);

/* 128-byte ncclUniqueId for world > 1 (call on rank 0, broadcast to all ranks).
 * NCCL is resolved at run time (dlopen); REFINE_E_NCCL if it is unavailable. */
refine_status refine_nccl_id(void* out128);

/* Host-only: the CSR halo plan of `rank` (no GPU needed; the multi-rank init uses
 * the same routine).  row_begin/row_end/col_lo/col_hi: every rank's rows and the
 * smallest/largest column its rows reference (world entries each).  A rank
 * receives the X rows [col_lo, row_begin) and [row_end, col_hi] it does not own,
 * stored in its halo buffer in that order.  send/recv: up to cap segments of 4
 * int64 {peer, first global row, row count, offset} (offset: local row for send,
 * halo row for recv); *nsend, *nrecv: segment counts; *halo_rows: halo size. */
int32_t refine_halo_plan(int32_t world, int32_t rank, const int64_t* row_begin, const int64_t* row_end,
                         const int64_t* col_lo, const int64_t* col_hi, int64_t* send, int32_t* nsend,
                         int64_t* recv, int32_t* nrecv, int64_t* halo_rows, int32_t cap);

/* Test hook: copy an intermediate of the LAST sweep to device buffer dst
 * (synchronises).  what: 0 W = A X^ - shift X^ (n_loc x k, for the sweep's un-flipped input), 1 sigma (k), 2 U (k x k,
 * un-flipped modified-LU factor), 3 Y_1 (k x k, unit lower), 4 T (k x k),
 * 5 dtilde (k), 6 alpha (k), 7 E_11 (k x k), 8 Y (n_loc x k, materialised by
 * the tall-skinny triangular apply Y_2 = X_2 U^{-1}; expects the sweep's input X
 * in dst on entry), 9 status-independent stats vector (8 doubles), 10 clock64 phase
 * log of the k x k kernels (REFINE_KXK_TIMING=1; 64 raw int64), 11 the CSR S1 kernel's
 * geometry (9 doubles: stencil SpMM on, tile R, L, column blocks, grid, grid nx, ny, nz,
 * gather rows per chunk). */
refine_status refine_debug_get(refine_ctx* c, int32_t what, double* dst);

#ifdef __cplusplus
}
#endif
#endif
