// refine.cu -- host runtime and C ABI (include/refine.h) of the B200-native refinement sweep.
//
// One sweep = the launch sequence below on the caller's stream:
//   dense: gemm_ax (DMMA, split-K) -> w_finish            | CSR: spmm_csr (fma chain, fused)
//   kxk_rq -> passB -> passB_reduce -> [join kxk_lu] kxk_finish -> passC -> norm_reduce -> normalize
//   (kxk_lu -- modified LU, T, U^{-1} of the top block -- needs only X^_1 and runs on a side stream)
// Device-side conditions are carried by a status word every kernel checks first, so a
// failed or halted sweep leaves X untouched and refine_run needs no per-sweep host sync.
//
// Row partition (world > 1): rank r owns rows [rb_r, re_r), rank 0 the
// top k x k block.  Per sweep: X exchange (dense: all-gather of X; CSR: halo rows) -> S1 ->
// all-gather of the alpha/g double-double vectors -> kxk_rq (identical d on every rank; kxk_lu on
// rank 0) -> passB -> all-gather of [M2 | G2 | rr2] -> kxk_finish on rank 0 -> broadcast of
// [Csig | scal | stats | status] -> passC -> all-gather of the column norm partials ->
// normalize.  Every cross-rank sum is formed from gathered per-rank values in rank order, so
// all ranks hold bit-identical k x k state.  Collectives are NCCL (one process per GPU) or, for
// tests on one device, device copies between emulated ranks ("loopback": world > 1 with
// nccl_id == NULL).
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <utility>
#include <vector>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <new>

#include "../../include/refine.h"
#include "common.cuh"
#include "gemm_dense.cuh"
#include "kxk.cuh"
#include "passes.cuh"
#include "spmm_csr.cuh"
#include "spmm_stencil.cuh"
#include "tc_passes.cuh"
#include "ozaki.cuh"
#include "nccl_dl.h"

using namespace rf;

namespace {

constexpr int ST_HALT_CONVERGED = 100;   // refine_run: device-side stop (converged)

struct RunState {   // device-resident refine_run bookkeeping
  int32_t done;     // sweeps completed
  int32_t guard;    // 1: stopped by the divergence guard (refine_run's rr_fallback continues from there)
  double hist[4];   // last corr norms (ring) for the divergence guard
};

// After each sweep of refine_run: convergence (||E_L||_F <= tol; or rel_resid <=
// resid_tol), divergence (non-finite; the growth guard), and the
// reorthogonalisation gate (gram_dev of the sweep's input > reorth_tol).
__device__ __forceinline__ void run_check_kernel_body(int* status, RunState* rs, const double* stats, double tol,
                                                      int window, double factor, double resid_tol, double reorth_tol,
                                                      int* gate) {
  if (gate) *gate = 1;
  griddep_wait();   // (programmatic dependent launch: the predecessor's writes are visible after this)
  if (*status != ST_OK) return;
  const double c = stats[1];
  const int t = rs->done;
  rs->done = t + 1;
  if (!isfinite(c)) { *status = ST_DIVERGED; return; }
  if (c <= tol || (resid_tol > 0.0 && stats[0] <= resid_tol)) { *status = ST_HALT_CONVERGED; return; }
  if (window > 0 && window <= 4 && t >= window && c >= factor * rs->hist[(t - window) & 3]) {
    *status = ST_DIVERGED;
    rs->guard = 1;
    return;
  }
  rs->hist[t & 3] = c;
  if (gate && reorth_tol > 0.0 && stats[6] > reorth_tol) *gate = ST_OK;
}
__global__ void run_check_kernel(int* status, RunState* rs, const double* stats, double tol, int window,
                                 double factor, double resid_tol, double reorth_tol, int* gate) {
  run_check_kernel_body(status, rs, stats, tol, window, factor, resid_tol, reorth_tol, gate);
}

// ||A - shift I||_inf row sums with Neumaier-compensated accumulation (the oracle's summation
// class, reading R4): each lane carries (s, c) over its strided columns, the 32 lane pairs are
// combined by compensated adds, so delta = c ||A|| u agrees with the oracle's to O(u) even at a tie.
struct Nsum { double s, c; };
RF_DEV void nsum_add(Nsum& a, double x) {
  const double t = a.s + x;
  a.c += (fabs(a.s) >= fabs(x)) ? (a.s - t) + x : (x - t) + a.s;
  a.s = t;
}
// refine_run as ONE graph launch (single rank): a conditional WHILE node whose body is one sweep
// (+ the gated reorthogonalisation) followed by this check; the loop continues while the status is
// OK and fewer than iters sweeps ran, so nothing is launched after convergence or divergence.
__global__ void run_cond_kernel(int* status, RunState* rs, const double* stats, double tol, int window,
                                double factor, double resid_tol, double reorth_tol, int* gate, int iters,
                                cudaGraphConditionalHandle h) {
  run_check_kernel_body(status, rs, stats, tol, window, factor, resid_tol, reorth_tol, gate);
  cudaGraphSetConditional(h, (*status == ST_OK && rs->done < iters) ? 1u : 0u);
}

__global__ void absrow_max_dense_kernel(const double* A, int64_t lda, int64_t n_loc, int64_t n, int64_t row0,
                                        double shift, double* out_rows) {
  const int lane = threadIdx.x & 31;
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = w; i < n_loc; i += nw) {
    Nsum s = {0.0, 0.0};
    for (int64_t l = lane; l < n; l += 32) {
      double a = A[i * lda + l];
      if (l == row0 + i) a -= shift;
      nsum_add(s, fabs(a));
    }
    for (int o = 16; o; o >>= 1) {
      const double os = __shfl_xor_sync(0xffffffffu, s.s, o), oc = __shfl_xor_sync(0xffffffffu, s.c, o);
      nsum_add(s, os);
      s.c += oc;
    }
    if (lane == 0) out_rows[i] = s.s + s.c;
  }
}
__global__ void absrow_max_csr_kernel(const int32_t* rp, const int32_t* ci, const double* v, int64_t n_loc,
                                      int64_t row0, double shift, double* out_rows) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_loc; i += (int64_t)gridDim.x * blockDim.x) {
    Nsum s = {0.0, 0.0};
    bool diag = false;
    for (int32_t p = rp[i]; p < rp[i + 1]; ++p) {
      double a = v[p];
      if (ci[p] == row0 + i) { a -= shift; diag = true; }
      nsum_add(s, fabs(a));
    }
    if (!diag) nsum_add(s, fabs(shift));
    out_rows[i] = s.s + s.c;
  }
}
__global__ void max_kernel(const double* x, int64_t n, double* out) {
  __shared__ double s[1024];
  double m = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) m = fmax(m, x[i]);
  s[threadIdx.x] = m;
  __syncthreads();
  for (int o = blockDim.x / 2; o; o >>= 1) {
    if (threadIdx.x < o) s[threadIdx.x] = fmax(s[threadIdx.x], s[threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = s[0];
}

__global__ void col_range_kernel(const int32_t* rp, const int32_t* ci, int64_t n_loc, unsigned long long* out) {
  unsigned long long lo = ~0ull, hi = 0ull;
  const int64_t p0 = rp[0], p1 = rp[n_loc];
  for (int64_t p = p0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < p1; p += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long c = (unsigned long long)ci[p];
    lo = c < lo ? c : lo;
    hi = c > hi ? c : hi;
  }
  atomicMin(out, lo);
  atomicMax(out + 1, hi);
}

// X <- X~ for Rayleigh-Ritz / QR steps with opts.normalize == 0, behind the status word (a failed
// or gate-closed step leaves X untouched, like every other kernel of the step)
__global__ void copy_gated_kernel(const int* status, double* __restrict__ X, const double* __restrict__ Xt, int64_t cnt) {
  griddep_wait();   // (programmatic dependent launch: the predecessor's writes are visible after this)
  if (*status != ST_OK) return;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += (int64_t)gridDim.x * blockDim.x)
    X[i] = Xt[i];
}

int pad_kp(int k) {
  int kp = 8;
  while (kp < k) kp *= 2;
  return kp;
}

}  // namespace

struct refine_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  int sms = 148;
  int64_t n = 0, n_loc = 0, row_begin = 0, row_end = 0;
  int k = 0, kp = 0;
  bool csr = false;
  const double* A = nullptr;
  int64_t lda = 0;
  const int32_t *rp = nullptr, *ci = nullptr;
  const double* val = nullptr;
  // CSR gather kernel (spmm_gather_kernel): rows per chunk (0 = not eligible -> vec / generic
  // kernel) and the precomputed gather offsets (owned; indexed by absolute CSR position)
  int gather_R = 0, gather_un = 8;
  bool gated = false;   // phase(): launch with ws.status -> ws.gate (refine_run reorthogonalisation)
  bool in_rr = false;   // phase(): a Rayleigh-Ritz / Cholesky-QR step (O(1) products: always FP64)
  double* bdiag = nullptr;   // NEXT-2 pass B: FP64 diagonal partials (sms x 2 kp), in the pool
  int4 spmm_ord = {0, 0, 0, 0};   // spmm_gather chunk order (spmm_csr.cuh chunk_of; x = 0: identity)
  // opts.emul (dense S1 on the INT8 tensor cores, ozaki.cuh): A slices (init), X slices (per sweep)
  int32_t *oz_e = nullptr, *oz_f = nullptr;
  double* oz_diag = nullptr;
  int8_t *oz_A = nullptr, *oz_X = nullptr;
  int oz_ns = 0;
  int64_t oz_nks = 0, oz_nrt = 0, oz_ks_per = 0;
  int32_t* xoff_buf = nullptr;
  const int32_t* xoff = nullptr;
  double shift = 0.0;
  refine_opts opts{};
  int rank = 0, world = 1;
  Ws ws{};
  void* pool = nullptr;
  size_t pool_bytes = 0;
  // dense GEMM launch
  int gemm_bm = 0, nsplit = 1;
  // TMA-fed dense S1 (gemm_ax_tma_kernel): A's tensor map (fixed at init), X's (cached per pointer)
  bool gemm_tma = false;
  int gemm_tbk = 16;            // K rows per TMA stage of the dense S1 (X^ box height)
  bool pdl = true;              // programmatic dependent launch of the sweep's kernels (launch_k)
  CUtensorMap tm_A{}, tm_X{};
  const double* tm_X_ptr = nullptr;
  // TMA-fed pass B at k = 128 (passB2_tma_kernel): X's map (cached per pointer) and W's (fixed)
  bool pb_tma = false;
  int pc_pp = 0;                 // k = 128: ping-pong pass C (1: 2 stages of 32 rows, 3: 3 stages of 24 rows)
  CUtensorMap tm_Xc{};
  const double* tm_Xc_ptr = nullptr;
  bool pb_pp = false;            // k = 128: ping-pong pass B (passB2_pp_kernel)            // k = 128: ping-pong pass C (passC_pp_kernel)
  CUtensorMap tm_Xb{}, tm_Wb{};
  const double* tm_Xb_ptr = nullptr;
  int64_t kchunk = 0;
  int gemm_gx = 0;
  int n_ag = 0, w_fin_grid = 0, spmm_grid = 0;
  int n_ag_cur = 0;             // alpha/g slots written by this sweep's S1 kernel (kxk_rq reduces them)
  bool wfuse = false;           // dense S1: split-K fix-up / shift / alpha-g in the GEMM (fused_finish), no w_finish
  int* gemm_cnt = nullptr;      // its per-row-tile arrival counters (in the pool)
  int s1_only = -1;             // opts.square at world > 1: phase 0 runs only product 0 / 1 (an exchange between)
  double* Tfull = nullptr;      // loopback, dense, opts.square: the gathered T = A X of all emulated ranks
  // stencil SpMM (spmm_stencil.cuh): geometry, packed row records (owned), X tensor map cache
  bool st_on = false;
  StencilGeo st_geo{};
  double* st_meta = nullptr;
  int st_grid = 0, st_smem = 0;
  CUtensorMap st_tm{};
  const double* st_tm_x = nullptr;
  int passb_grid_y = 0, passc_grid = 0;
  RunState* run = nullptr;
  refine_status sticky = REFINE_OK;
  // graph
  bool use_graph = false;
  cudaGraphExec_t gexec = nullptr;
  double* gX = nullptr;
  cudaStream_t cap_stream = nullptr;   // graphs are captured on a private stream (the caller's may be legacy)
  cudaStream_t side = nullptr;         // kxk_lu (depends on X only) overlaps S1 / S2 / passB here
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // host-buffer entry point
  double* dX = nullptr;
  // refine_sweep_host's overlapped upload (dense, TMA GEMM): X^ in chunks on the h2d stream, each chunk
  // flagged by a 4-byte copy of the call's epoch into h2d_ready[chunk]; S1 starts on the first chunk
  cudaStream_t h2d = nullptr;
  cudaEvent_t ev_h2d = nullptr, ev_pre = nullptr;
  unsigned* h2d_ready = nullptr;       // device, H2D_MAX_CHUNKS flags
  unsigned* h2d_epoch_host = nullptr;  // pinned: the value the flag copies carry
  unsigned h2d_epoch = 0;
  int h2d_rows = 0;
  bool h2d_on = false;
  int launches = 0;
  // live per-kernel timing (refine_profile_begin/end): events at every kernel boundary
  cudaEvent_t* prof_ev = nullptr;
  int prof_cap = 0, prof_used = 0, prof_per_sweep = 0, prof_sweeps = 0, prof_max_sweeps = 0;
  // row partition
  bool loopback = false;                      // parent of `world` emulated ranks on one device
  bool loopback_kid = false;                  // one emulated rank (its X rows alias the parent's X)
  bool multi = false;                         // multi-rank code path (world > 1, or NCCL forced at world 1)
  std::vector<refine_ctx*> kids;
  ncclComm_t comm = nullptr;
  std::vector<int64_t> rb_all, re_all;        // every rank's rows
  double* Xfull = nullptr;                    // dense world > 1: gathered X (n x k)
  bool own_xfull = false;
  struct Seg { int peer; int64_t row, cnt, off; };   // rows [row, row + cnt); off = local / halo row
  std::vector<Seg> hsend, hrecv;
  double* bc = nullptr;                       // [Csig | scal | stats(8) | status] broadcast from rank 0
  size_t bc_cnt = 0;
  void mark() {
    if (prof_ev && prof_used < prof_cap) cudaEventRecord(prof_ev[prof_used++], stream);
  }
};

static refine_status cuda_fail(refine_ctx* c, cudaError_t e, const char* what) {
  if (e == cudaSuccess) return REFINE_OK;
  fprintf(stderr, "[refine] CUDA error in %s: %s\n", what, cudaGetErrorString(e));
  if (c) c->sticky = (e == cudaErrorMemoryAllocation) ? REFINE_E_NOMEM : REFINE_E_CUDA;
  return (e == cudaErrorMemoryAllocation) ? REFINE_E_NOMEM : REFINE_E_CUDA;
}
#define RF_CK(c, expr)                                          \
  do {                                                          \
    cudaError_t e_ = (expr);                                    \
    if (e_ != cudaSuccess) return cuda_fail((c), e_, #expr);    \
  } while (0)

// Launch with programmatic dependent launch (PDL) when pdl: the kernel may be scheduled while its
// stream predecessor drains and waits in griddep_wait() -- the sweep is a chain of short kernels whose
// launch latency otherwise sits between every pair (REFINE_PDL=0 disables it).
template <typename... KArgs, typename... Args>
static cudaError_t launch_k(bool pdl, void (*kern)(KArgs...), dim3 g, dim3 b, size_t smem, cudaStream_t s,
                            Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = g;
  cfg.blockDim = b;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = pdl ? at : nullptr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// ---------------------------------------------------------------- per-KP kernel tables
template <int KP> struct Tiles;
//                 GEMM: BM  WM  WN  BK  ST | passB: TA  TB  WA WB  BR | passC: NC BM WM WN
template <> struct Tiles<8>   { static constexpr int G[5] = {64, 16, 8, 32, 4};   static constexpr int B[5] = {8, 16, 1, 2, 32};   static constexpr int C[4] = {8, 64, 8, 1}; };
template <> struct Tiles<16>  { static constexpr int G[5] = {64, 16, 16, 32, 4};  static constexpr int B[5] = {16, 32, 2, 4, 32};  static constexpr int C[4] = {16, 64, 8, 1}; };
template <> struct Tiles<32>  { static constexpr int G[5] = {128, 32, 16, 32, 2}; static constexpr int B[5] = {32, 64, 1, 4, 32};  static constexpr int C[4] = {32, 64, 4, 2}; };
template <> struct Tiles<64>  { static constexpr int G[5] = {128, 64, 16, 32, 2}; static constexpr int B[5] = {64, 128, 2, 4, 16}; static constexpr int C[4] = {64, 64, 2, 4}; };
template <> struct Tiles<128> { static constexpr int G[5] = {64, 32, 32, 32, 2};  static constexpr int B[5] = {64, 64, 2, 2, 16};  static constexpr int C[4] = {128, 32, 2, 8}; };

// ---------------------------------------------------------------- stencil SpMM (spmm_stencil.cuh)
static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static void* fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
  }
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
}

// 4-D view {k, nx, ny, nz} of the row-major n x k block X, box {KC, R + 2, L + 2 hy, 1}
static bool stencil_tensor_map(refine_ctx* c, const double* X) {
  if (c->st_tm_x == X) return true;
  auto enc = tensor_map_encoder();
  if (!enc) return false;
  const StencilGeo& g = c->st_geo;
  const cuuint64_t K = (cuuint64_t)c->k;
  cuuint64_t dims[4] = {K, (cuuint64_t)g.nx, (cuuint64_t)g.ny, (cuuint64_t)g.nz};
  cuuint64_t strides[3] = {K * 8, K * 8 * g.nx, K * 8 * g.nx * g.ny};
  cuuint32_t box[4] = {(cuuint32_t)g.KC, (cuuint32_t)g.Rb, (cuuint32_t)g.Lb, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = enc(&c->st_tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(X), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return false;
  c->st_tm_x = X;
  return true;
}

// dense S1 tensor maps: 2-D {cols, rows} views, 16-double boxes with the 128-byte swizzle
static bool encode_2d(CUtensorMap* m, const double* base, uint64_t cols, uint64_t rows, uint64_t ld, uint32_t box_rows) {
  auto enc = tensor_map_encoder();
  if (!enc || ((uintptr_t)base % 16) != 0 || (ld * 8) % 16 != 0) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld * 8};
  cuuint32_t box[2] = {16, box_rows};
  cuuint32_t es[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
static int PB2_TMA_WAVES = getenv("REFINE_PB2_WAVES") ? atoi(getenv("REFINE_PB2_WAVES")) : 2;   // (1 / 2 / 3 measured within 0.5 %)
static bool passb_x_map(refine_ctx* c, const double* X) {   // local X rows -> boxes of 16 rows x 16 columns
  if (c->tm_Xb_ptr == X) return true;
  if (!encode_2d(&c->tm_Xb, X, (uint64_t)c->k, (uint64_t)c->n_loc, (uint64_t)c->k, PassB2TmaCfg<128>::BR)) return false;
  c->tm_Xb_ptr = X;
  return true;
}
static bool passc3_x_map(refine_ctx* c, const double* X, int rows) {   // local X rows -> boxes of `rows` x 16 columns
  if (c->tm_Xc_ptr == X) return true;
  if (!encode_2d(&c->tm_Xc, X, (uint64_t)c->k, (uint64_t)c->n_loc, (uint64_t)c->k, rows)) return false;
  c->tm_Xc_ptr = X;
  return true;
}
static bool gemm_x_map(refine_ctx* c, const double* X) {   // X (n x k) -> boxes of 16 (K rows) x 16 columns
  if (c->tm_X_ptr == X) return true;
  if (!encode_2d(&c->tm_X, X, (uint64_t)c->k, (uint64_t)c->n, (uint64_t)c->k, (uint32_t)c->gemm_tbk)) return false;
  c->tm_X_ptr = X;
  return true;
}

template <int KC, int NZR>
static void stencil_kernel_launch(refine_ctx* c, const Ws& ws) {
  if (ws.shift != 0.0)
    launch_k(c->pdl, spmm_stencil_kernel<KC, NZR, true>, dim3(c->st_grid), dim3(ST_BLOCK), c->st_smem, c->stream, ws,
             c->st_tm, (const double*)c->st_meta, c->st_geo);
  else
    launch_k(c->pdl, spmm_stencil_kernel<KC, NZR, false>, dim3(c->st_grid), dim3(ST_BLOCK), c->st_smem, c->stream, ws,
             c->st_tm, (const double*)c->st_meta, c->st_geo);
}
static bool stencil_launch(refine_ctx* c, const double* X, const Ws& ws) {
  if (!stencil_tensor_map(c, X)) return false;
  const int kc = c->st_geo.KC, nzr = c->st_geo.nzr;
  if (kc == 32) nzr == 5 ? stencil_kernel_launch<32, 5>(c, ws) : stencil_kernel_launch<32, 7>(c, ws);
  else if (kc == 16) nzr == 5 ? stencil_kernel_launch<16, 5>(c, ws) : stencil_kernel_launch<16, 7>(c, ws);
  else nzr == 5 ? stencil_kernel_launch<8, 5>(c, ws) : stencil_kernel_launch<8, 7>(c, ws);
  return true;
}

// Detect a 2-D / 3-D grid stencil in the CSR (every nonzero offset in {0, +-1, +-d2, +-d3}, no
// wrap across lines / planes, <= 7 nonzeros per row), pick the tile, pack the row records and size
// the persistent grid.  Single rank, not the squared operator.  REFINE_SPMM=gather disables it.
static cudaError_t stencil_setup(refine_ctx* c) {
  c->st_on = false;
  const char* env = getenv("REFINE_SPMM");
  const bool force = env && strcmp(env, "stencil") == 0;
  if ((env && strcmp(env, "gather") == 0) || !c->csr || c->multi || c->opts.square) return cudaSuccess;
  const int k = c->k;
  const int KC = (k % 32 == 0) ? 32 : (k % 16 == 0) ? 16 : (k % 8 == 0) ? 8 : 0;
  if (KC == 0 || k > KMAX) return cudaSuccess;
  const int64_t n = c->n_loc;
  std::vector<int32_t> rp(n + 1);
  cudaError_t e = cudaMemcpy(rp.data(), c->rp, (n + 1) * sizeof(int32_t), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return e;
  const int64_t nnz = (int64_t)rp[n] - rp[0];
  if (nnz <= 0 || rp[0] != 0) return cudaSuccess;
  std::vector<int32_t> ci(nnz);
  if ((e = cudaMemcpy(ci.data(), c->ci, nnz * sizeof(int32_t), cudaMemcpyDeviceToHost)) != cudaSuccess) return e;
  std::vector<int64_t> lv;   // distinct nonzero |offsets|
  for (int64_t i = 0; i < n; ++i)
    for (int32_t p = rp[i]; p < rp[i + 1]; ++p) {
      const int64_t o = std::llabs((int64_t)ci[p] - i);
      if (o == 0 || std::find(lv.begin(), lv.end(), o) != lv.end()) continue;
      if (lv.size() == 3) return cudaSuccess;   // not a 2-D / 3-D axis stencil
      lv.push_back(o);
    }
  std::sort(lv.begin(), lv.end());
  if (getenv("REFINE_VERBOSE")) {
    fprintf(stderr, "[refine] stencil offsets:");
    for (auto v : lv) fprintf(stderr, " %lld", (long long)v);
    fprintf(stderr, "\n");
  }
  StencilGeo g{};
  int64_t chk_d2, chk_d3;
  if (lv.size() == 3 && lv[0] == 1 && lv[2] % lv[1] == 0 && n % lv[2] == 0) {          // 3-D
    g.nx = (int)lv[1]; g.ny = (int)(lv[2] / lv[1]); g.nz = (int)(n / lv[2]);
    g.d2 = lv[1]; g.d3 = lv[2]; g.hy = 1;
    chk_d2 = lv[1]; chk_d3 = lv[2];
  } else if (lv.size() == 2 && lv[0] == 1 && n % lv[1] == 0) {                            // 2-D: swept along y
    g.nx = (int)lv[1]; g.ny = 1; g.nz = (int)(n / lv[1]);
    g.d2 = 0; g.d3 = lv[1]; g.hy = 0;
    chk_d2 = lv[1]; chk_d3 = lv[1];
  } else {
    return cudaSuccess;
  }
  if (g.nx < 2 || g.nz < 1 || g.d3 * (int64_t)k >= INT32_MAX) return cudaSuccess;   // (32-bit in-plane W offsets)
  // default: 3-D grids with k >= 64 (cfg5: 1.91 vs 2.31 ms for the gather kernel) and 2-D grids with
  // k a multiple of 32 (cfg4: 0.123 vs 0.148 ms, once a CTA owns whole 128-point line segments at one
  // CTA per SM and the slabs are split evenly -- 64-point segments at two CTAs per SM measured 0.173 ms).
  // REFINE_SPMM=stencil forces it wherever the structure allows (tests).
  if (!force && !(g.hy ? k >= 64 : k % 32 == 0)) return cudaSuccess;
  int* dflag = nullptr;
  if ((e = cudaMalloc(&dflag, 2 * sizeof(int))) != cudaSuccess) return e;
  cudaMemsetAsync(dflag, 0, 2 * sizeof(int), c->stream);
  stencil_check_kernel<<<c->sms * 4, 256, 0, c->stream>>>(c->rp, c->ci, n, g.nx, chk_d2, chk_d3, dflag);
  int hf[2] = {1, 0};
  e = cudaMemcpyAsync(hf, dflag, sizeof(hf), cudaMemcpyDeviceToHost, c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  cudaFree(dflag);
  if (e != cudaSuccess) return e;
  if (getenv("REFINE_VERBOSE"))
    fprintf(stderr, "[refine] stencil check: grid %d x %d x %d, violations %d, max row %d\n", g.nx, g.ny, g.nz, hf[0],
            hf[1]);
  if (hf[0] != 0 || hf[1] > 7) return cudaSuccess;
  g.nzr = hf[1] <= 5 ? 5 : 7;
  g.KC = KC;
  g.nq = k / KC;
  // tile: maximise the staged-row reuse L R / ((L + 2 hy)(R + 2)) times the tile utilisation,
  // 4 slots within the shared-memory budget of one CTA per SM (two per SM, i.e. half-size tiles and one
  // row per thread per slab, measured 40 % slower on the 2-D cfg4: the per-slab overhead dominates)
  const int occ = getenv("REFINE_ST_OCC") ? atoi(getenv("REFINE_ST_OCC")) : 1;
  const int budget = (occ == 1 ? 220 : 110) * 1024 - 128;
  const int Ls3[] = {1, 2, 4, 5, 8, 10, 16}, Rs[] = {8, 16, 20, 24, 32, 40, 48, 64, 96, 128, 192};
  double best = -1.0;
  for (int L : Ls3) {
    if (!g.hy && L != 1) continue;
    for (int R : Rs) {
      const int Rb = R + 2, Lb = L + 2 * g.hy;
      const int box = KC * Rb * Lb * 8, meta = L * R * (g.nzr + 1) * 8;
      const int slot = (box + meta + 127) & ~127;
      if (ST_SLOTS * slot + 128 > budget || R > 2 * g.nx) continue;
      const int ntx = (g.nx + R - 1) / R, nty = (g.ny + L - 1) / L;
      const double util = (double)g.nx / (ntx * R) * ((double)g.ny / (nty * L));
      const double score = (double)(L * R) / (Lb * Rb) * util;
      if (score > best + 1e-9) {
        best = score;
        g.R = R; g.L = L; g.Rb = Rb; g.Lb = Lb; g.ntx = ntx; g.nty = nty;
        g.box_bytes = box; g.meta_bytes = meta; g.slot_bytes = slot;
      }
    }
  }
  if (best <= 0.0) return cudaSuccess;
  const int sms = (c->rank == 0 && c->sms > 1) ? c->sms - 1 : c->sms;   // one SM left to kxk_lu
  const int nb = std::max(1, sms * occ / g.nq);
  const int64_t pencils = (int64_t)g.ntx * g.nty;
  int nseg = (int)std::min<int64_t>(g.nz, std::max<int64_t>(1, (8 * (int64_t)nb + pencils - 1) / pencils));
  g.zlen = (g.nz + nseg - 1) / nseg;
  g.nseg = (g.nz + g.zlen - 1) / g.zlen;
  g.blocks = (int64_t)g.ntx * g.nty * g.nz;
  {  // alpha / g FP64 blocks of at most 32 rows per thread (rows per thread per slab: L R / rows per pass),
     // then double-double: 8 / 16 / 32 rows measured 1.930 / 1.913 / 1.906 ms at cfg5 (the merge shuffles);
     // a block's same-sign x_ij^2 (or x_ij w_ij ~ d_j x_ij^2) terms carry <= 31 u / 2 of its own sum
    const int rgp = ST_THREADS / (KC >= 16 ? 8 : KC / 2);
    const int rpt = (g.L * g.R + rgp - 1) / rgp;
    g.mrg = std::max(1, (getenv("REFINE_ST_ROWS") ? atoi(getenv("REFINE_ST_ROWS")) : 32) / rpt);
  }
  const size_t meta_bytes = (size_t)g.blocks * g.meta_bytes;
  if ((e = cudaMalloc(&c->st_meta, meta_bytes)) != cudaSuccess) return e;
  cudaMemsetAsync(c->st_meta, 0, meta_bytes, c->stream);
  if (g.nzr == 5) stencil_pack_kernel<5><<<c->sms * 8, 256, 0, c->stream>>>(c->rp, c->ci, c->val, g, c->st_meta);
  else stencil_pack_kernel<7><<<c->sms * 8, 256, 0, c->stream>>>(c->rp, c->ci, c->val, g, c->st_meta);
  if (g.nzr == 5) stencil_flag_kernel<5><<<c->sms * 4, 128, 0, c->stream>>>(g, c->st_meta);
  else stencil_flag_kernel<7><<<c->sms * 4, 128, 0, c->stream>>>(g, c->st_meta);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  c->st_geo = g;
  c->st_grid = nb * g.nq;
  c->st_smem = std::max(ST_SLOTS * g.slot_bytes + 128, 128 + 8 * ST_THREADS * 16);   // (+ the final dd reduction)
  auto attr = [&](auto kern) { return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, c->st_smem); };
  for (int sh = 0; sh < 2 && e == cudaSuccess; ++sh) {
    if (KC == 32) e = g.nzr == 5 ? (sh ? attr(spmm_stencil_kernel<32, 5, true>) : attr(spmm_stencil_kernel<32, 5, false>))
                                 : (sh ? attr(spmm_stencil_kernel<32, 7, true>) : attr(spmm_stencil_kernel<32, 7, false>));
    else if (KC == 16) e = g.nzr == 5 ? (sh ? attr(spmm_stencil_kernel<16, 5, true>) : attr(spmm_stencil_kernel<16, 5, false>))
                                      : (sh ? attr(spmm_stencil_kernel<16, 7, true>) : attr(spmm_stencil_kernel<16, 7, false>));
    else e = g.nzr == 5 ? (sh ? attr(spmm_stencil_kernel<8, 5, true>) : attr(spmm_stencil_kernel<8, 5, false>))
                        : (sh ? attr(spmm_stencil_kernel<8, 7, true>) : attr(spmm_stencil_kernel<8, 7, false>));
  }
  if (e != cudaSuccess) return e;
  c->st_on = tensor_map_encoder() != nullptr;
  if (getenv("REFINE_VERBOSE"))
    fprintf(stderr, "[refine] stencil SpMM %s: tile R %d L %d, KC %d x %d, grid %d, segments %d x %d, slot %d B x %d\n",
            c->st_on ? "on" : "off (no tensor-map encoder)", g.R, g.L, g.KC, g.nq, c->st_grid, g.nseg, g.zlen,
            g.slot_bytes, ST_SLOTS);
  return cudaSuccess;
}

// Xg: the rows gathered (X, or A X for the second product of the squared operator), Xo: own rows
template <bool HALO>
static void launch_spmm(refine_ctx* c, bool vec, const double* Xg, const double* Xo, const Ws& ws) {
  cudaStream_t s = c->stream;
  const int g = c->spmm_grid;
  c->n_ag_cur = g;                // the gather / per-row kernels write one slot per CTA
  if (!HALO && c->st_on && Xg == Xo && ((uintptr_t)Xg % 16) == 0 && stencil_launch(c, Xg, ws)) {
    c->n_ag_cur = c->st_grid / c->st_geo.nq;
    return;
  }
  if (vec && c->gather_R > 0) {   // vec: 16-byte aligned X / halo rows
    const int R = c->gather_R;
    const int4 ord = HALO ? make_int4(0, 0, 0, 0) : c->spmm_ord;
    auto go = [&](auto kern) { launch_k(c->pdl, kern, dim3(g), dim3(256), 0, s, ws, c->rp, c->xoff, c->val, Xg, R, Xo, ord); };
#define RF_GATHER_K(KK)                                                          \
  case KK:                                                                       \
    if (c->gather_un == 5) go(spmm_gather_kernel<KK, HALO, 5>);                  \
    else if (c->gather_un == 7) go(spmm_gather_kernel<KK, HALO, 7>);             \
    else go(spmm_gather_kernel<KK, HALO, 8>);                                    \
    break;
    switch (c->k) {
      RF_GATHER_K(2)
      RF_GATHER_K(4)
      RF_GATHER_K(8)
      RF_GATHER_K(16)
      RF_GATHER_K(32)
      RF_GATHER_K(64)
      default: RF_GATHER_K(128)
    }
#undef RF_GATHER_K
    return;
  }
  if (vec) {
    switch (c->k) {
      case 2: spmm_csr_vec_kernel<1, 1, HALO><<<g, 256, 0, s>>>(ws, c->rp, c->ci, c->val, Xo, Xg); break;
      case 4: spmm_csr_vec_kernel<1, 2, HALO><<<g, 256, 0, s>>>(ws, c->rp, c->ci, c->val, Xo, Xg); break;
      case 8: spmm_csr_vec_kernel<1, 4, HALO><<<g, 256, 0, s>>>(ws, c->rp, c->ci, c->val, Xo, Xg); break;
      case 16: spmm_csr_vec_kernel<1, 8, HALO><<<g, 256, 0, s>>>(ws, c->rp, c->ci, c->val, Xo, Xg); break;
      case 32: spmm_csr_vec_kernel<1, 16, HALO><<<g, 256, 0, s>>>(ws, c->rp, c->ci, c->val, Xo, Xg); break;
      case 64: spmm_csr_vec_kernel<1, 32, HALO><<<g, 256, 0, s>>>(ws, c->rp, c->ci, c->val, Xo, Xg); break;
      default: spmm_csr_vec_kernel<2, 32, HALO><<<g, 256, 0, s>>>(ws, c->rp, c->ci, c->val, Xo, Xg); break;
    }
  } else {
    switch ((c->k + 31) / 32) {
      case 1: spmm_csr_kernel<1, HALO><<<g, 256, 0, s>>>(ws, c->rp, c->ci, c->val, Xo, Xg); break;
      case 2: spmm_csr_kernel<2, HALO><<<g, 256, 0, s>>>(ws, c->rp, c->ci, c->val, Xo, Xg); break;
      case 3: spmm_csr_kernel<3, HALO><<<g, 256, 0, s>>>(ws, c->rp, c->ci, c->val, Xo, Xg); break;
      default: spmm_csr_kernel<4, HALO><<<g, 256, 0, s>>>(ws, c->rp, c->ci, c->val, Xo, Xg); break;
    }
  }
}

// kxk_finish as one thread-block cluster of kxk_cluster(k) CTAs (16 for k > 64 when the device can
// schedule a non-portable 16-CTA cluster of this kernel: checked once; REFINE_KXK_CL16=0 keeps 8)
static bool kxk_allow16() {
  const char* e = getenv("REFINE_KXK_CL16");   // (read per launch: tests switch it within one process)
  if (e && e[0] == '0') return false;
  static int ok = -1;
  if (ok < 0) {
    ok = 0;
    if (cudaFuncSetAttribute(kxk_finish_kernel<false>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(16, 1, 1);
      cfg.blockDim = dim3(KXK_THREADS, 1, 1);
      cfg.dynamicSmemBytes = FK_SMEM * 8;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 16;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int nc = 0;
      if (cudaOccupancyMaxActiveClusters(&nc, kxk_finish_kernel<false>, &cfg) == cudaSuccess && nc >= 1) ok = 1;
    }
    cudaGetLastError();
  }
  return ok == 1;
}
static cudaError_t launch_kxk_finish(const Ws& ws, double* X, cudaStream_t s, bool pdl) {
  static const bool no_small = getenv("REFINE_KXK_SMALL") && getenv("REFINE_KXK_SMALL")[0] == '0';
  if (ws.k <= KXK_SMALL && !no_small)   // one CTA, everything in shared memory
    return launch_k(pdl, kxk_finish_kernel<true>, dim3(1), dim3(KXK_THREADS), kxk_small_smem_doubles(ws.k) * 8, s, ws,
                    X, (const double*)ws.W);
  const int ncl = kxk_cluster(ws.k, kxk_allow16());
  if (ncl == 1)   // (a plain launch is an implicit 1-CTA cluster)
    return launch_k(pdl, kxk_finish_kernel<false>, dim3(1), dim3(KXK_THREADS), FK_SMEM * 8, s, ws, X,
                    (const double*)ws.W);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ncl, 1, 1);
  cfg.blockDim = dim3(KXK_THREADS, 1, 1);
  cfg.dynamicSmemBytes = FK_SMEM * 8;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = ncl;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, kxk_finish_kernel<false>, ws, X, (const double*)ws.W);
}

template <int KP>
struct Kern {
  using TT = Tiles<KP>;
  static constexpr int GBM = TT::G[0], GWM = TT::G[1], GWN = TT::G[2], GBK = TT::G[3], GST = TT::G[4];
  static constexpr int BTA = TT::B[0], BTB = TT::B[1], BWA = TT::B[2], BWB = TT::B[3], BBR = TT::B[4];
  static constexpr int CNC = TT::C[0], CBM = TT::C[1], CWM = TT::C[2], CWN = TT::C[3];
  using GC = GemmCfg<KP, GBM, GWM, GWN, GBK, GST>;
  using BC = PassBCfg<KP, BTA, BTB, BWA, BWB, BBR>;
  using CC = PassCCfg<KP, CNC, CBM, CWM, CWN>;
  static constexpr auto gemm = gemm_ax_kernel<KP, GBM, GWM, GWN, GBK, GST>;
  // TMA-fed S1 (KP >= 16): BK = 16 K-steps in a TST-deep ring, the cp.async kernel's warp tiles
  static constexpr bool TMA_OK = KP >= 16;
  static constexpr int TBK = 16, TST = 4;   // (k = 16 measured: 32-row stages 35.0 us, 8 stages 35.5 us, this 31 us)
  using TGC = GemmCfg<KP, GBM, GWM, GWN, TBK, TST>;
  static constexpr int T_SMEM = gemm_tma_smem<(KP >= 16 ? KP : 16), GBM, TBK, TST>();
  static constexpr auto gemm_tma = gemm_ax_tma_kernel<(KP >= 16 ? KP : 16), GBM, GWM, (KP >= 16 ? GWN : 16), TBK, TST>;
  // k = 128: pass B2 (all-a CTA tiles, balanced 7-unit grid); smaller k: the 2-D tiled pass B
  // (measured faster there: cfg4 0.19 vs 0.22 ms, cfg3 0.034 vs 0.039 ms)
  static constexpr bool B2 = KP >= 128;
  using B2C = PassB2Cfg<(KP >= 32 ? KP : 32)>;
  static constexpr auto passB = B2 ? (decltype(&passB_kernel<KP, BTA, BTB, BWA, BWB, BBR>))passB2_kernel<(KP >= 32 ? KP : 32)>
                                   : passB_kernel<KP, BTA, BTB, BWA, BWB, BBR>;
  static constexpr auto passBred = B2 ? (decltype(&passB_reduce_kernel<KP, BTA, BTB, BWA, BWB, BBR>))passB2_reduce_kernel<(KP >= 32 ? KP : 32)>
                                      : passB_reduce_kernel<KP, BTA, BTB, BWA, BWB, BBR>;
  static constexpr int B_THREADS = B2 ? B2C::THREADS : BC::THREADS;
  static constexpr int B_SMEM = B2 ? B2C::SMEM : BC::SMEM;
  static constexpr int B_NT = B2 ? B2C::NT : BC::NTILES;
  static constexpr size_t B_TILE = B2 ? (size_t)B2C::TA * B2C::TB : (size_t)BTA * BTB;
  static constexpr auto passC = passC_kernel<KP, CNC, CBM, CWM, CWN, true>;       // RR / QR steps (norm sums)
  static constexpr auto passC_sweep = passC_kernel<KP, CNC, CBM, CWM, CWN, false>; // a sweep (norms folded earlier)
  static constexpr int TKP = KP >= 32 ? KP : 32;   // tcgen05 passes (NEXT-2) exist for KP >= 32
  static_assert(CNC == KP, "pass C writes X in place: one CTA must own whole rows (all k columns)");

  static cudaError_t setup(refine_ctx* c) {
    cudaError_t e;
    if ((e = cudaFuncSetAttribute(gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, GC::SMEM))) return e;
    if ((e = cudaFuncSetAttribute(passB, cudaFuncAttributeMaxDynamicSharedMemorySize, B_SMEM))) return e;
    if ((e = cudaFuncSetAttribute(passC, cudaFuncAttributeMaxDynamicSharedMemorySize, CC::SMEM))) return e;
    if ((e = cudaFuncSetAttribute(passC_sweep, cudaFuncAttributeMaxDynamicSharedMemorySize, CC::SMEM))) return e;
    if (KP == 128 && c->opts.emul)   // pass C on the INT8 tensor cores (ozaki.cuh)
      if ((e = cudaFuncSetAttribute(passC_oz_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, OZC_SMEM))) return e;
    if (KP >= 32 && c->opts.mixed) {   // NEXT-2 tcgen05 passes (tc_passes.cuh)
      if ((e = cudaFuncSetAttribute(passB_tc_kernel<TKP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    TcbCfg<TKP>::SMEM))) return e;
      if ((e = cudaFuncSetAttribute(passC_tc_kernel<TKP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    TccCfg<TKP>::SMEM))) return e;
    }
    int occ = 1;
    // dense GEMM: split-K so the grid fills whole waves of resident CTAs
    if (!c->csr) {
      if (c->gemm_tma && TMA_OK) {
        c->gemm_tbk = TBK;
        if ((e = cudaFuncSetAttribute(gemm_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, T_SMEM))) return e;
        if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, gemm_tma, TGC::THREADS + 32, T_SMEM))) return e;
      } else {
        c->gemm_tma = false;
        if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, gemm, GC::THREADS, GC::SMEM))) return e;
      }
      occ = std::max(occ, 1);
      const int slots = c->sms * occ;
      c->gemm_bm = GBM;
      c->gemm_gx = (int)((c->n_loc + GBM - 1) / GBM);
      const int64_t kiters = (c->n + GBK - 1) / GBK;
      // split-K: smallest split whose grid fills >= 3 waves of resident CTAs at >= 90% wave
      // efficiency (each extra split adds 2 x n_loc x k x 8 bytes of partial traffic)
      int best = 1;
      double best_eff = -1.0;
      for (int s = 1; s <= 16 && s <= kiters; ++s) {
        const int64_t ctas = (int64_t)c->gemm_gx * s;
        const double waves = std::ceil((double)ctas / slots);
        double eff = (double)ctas / (waves * slots);
        if (ctas < 3 * slots) eff *= (double)ctas / (3.0 * slots);
        if (eff > best_eff + 0.02) { best_eff = eff; best = s; }
        if (eff >= 0.9 && ctas >= 3 * slots) break;
      }
      if (getenv("REFINE_NSPLIT")) best = std::max(1, std::min<int>(atoi(getenv("REFINE_NSPLIT")), (int)kiters));   // (measurements)
      c->nsplit = best;
      const int64_t kit = (kiters + best - 1) / best;
      c->kchunk = kit * GBK;
      c->nsplit = (int)((c->n + c->kchunk - 1) / c->kchunk);
    }
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, passB, B_THREADS, B_SMEM))) return e;
    occ = std::max(occ, 1);
    const int64_t rows = std::max<int64_t>(c->n_loc - c->ws.top, 1);
    static const int64_t pb_min_rows = getenv("REFINE_PB_MINROWS") ? std::max(32, atoi(getenv("REFINE_PB_MINROWS"))) : 64;
    const int64_t max_chunks = std::max<int64_t>((rows + pb_min_rows - 1) / pb_min_rows, 1);   // >= pb_min_rows rows per chunk
    c->passb_grid_y = (int)std::min<int64_t>(std::max(c->sms * occ / B_NT, 1), max_chunks);
    if (B2 && B2C::PAIRED) {   // 7 balanced units per pair of chunks (passB2_kernel / passB2_tma_kernel)
      if (c->pb_tma) {   // one CTA per SM: one wave of units
        if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, passB2_tma_kernel<128>, PassB2TmaCfg<128>::THREADS + 32,
                                                               PassB2TmaCfg<128>::SMEM))) return e;
        occ = std::max(occ, 1) * PB2_TMA_WAVES;
      }
      const int pairs = (int)std::max<int64_t>(1, std::min<int64_t>(c->sms * occ / 7, std::max<int64_t>(max_chunks / 2, 1)));
      c->passb_grid_y = 2 * pairs;
    }
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, passC, CC::THREADS, CC::SMEM))) return e;
    occ = std::max(occ, 1);
    const int64_t ctiles = std::max<int64_t>((rows + CBM - 1) / CBM, 1);
    c->passc_grid = (int)std::min<int64_t>(std::max(c->sms * occ / (KP / CNC), 1), ctiles);
    return cudaSuccess;
  }

  static void sizes(refine_ctx* c, size_t& bpart, size_t& brr, size_t& nslot) {
    // the tcgen05 passes (opts.mixed) write one partial per SM in the same slot layouts
    const bool tc = KP >= 32 && c->opts.mixed;
    const size_t cb = tc ? std::max(c->passb_grid_y, c->sms) : c->passb_grid_y;
    const size_t cc = (tc || c->opts.emul) ? std::max(c->passc_grid, c->sms) : c->passc_grid;
    bpart = std::max(cb * B_NT * B_TILE, tc ? (size_t)c->sms * 2 * KP * KP : 0);   // (tc: passB2 slot layout)
    brr = cb * KP;
    nslot = cc * KP;
  }
  // NEXT-2: this sweep's passes B and C on tcgen05 (k a multiple of 16 in [32, 128], not a
  // Rayleigh-Ritz / QR step, 16-byte aligned X for the bulk copies)
  static bool use_tc(const refine_ctx* c, const double* X) {
    return KP >= 32 && c->opts.mixed && c->k % 16 == 0 && !c->in_rr && ((uintptr_t)X % 16 == 0);
  }
  // pass C on tcgen05 only where the FP64 pass is compute bound: 2k^2 flop vs 24k bytes per row
  // crosses over at k ~ 68 on this part (DMMA 37 TFLOP/s, HBM 6.5 TB/s), so k <= 64 keeps the
  // FP64 pass C (already at the HBM roofline); opts.mixed = 2 forces it (tests, measurements)
  static bool use_tc_c(const refine_ctx* c, const double* X) {
    return use_tc(c, X) && (c->k > 64 || c->opts.mixed >= 2);
  }

  // phase ph of one sweep on this rank (see the file header); returns kernels launched
  static int phase(refine_ctx* c, int ph, double* X) {
    Ws ws = c->ws;
    if (c->gated) ws.status = ws.gate;     // refine_run's reorthogonalisation pipeline runs behind the gate
    cudaStream_t s = c->stream;
    int n = 0;
    const bool xv16 = (c->k % 2 == 0) && ((uintptr_t)X % 16 == 0);
    switch (ph) {
      case 0:    // S1 (+ S2 partials); S3 (kxk_lu, X^_1 only) forked onto the side stream
      case 10: {  // Rayleigh-Ritz: S1 only (W = (A - shift I) X)
        if (ph == 0 && ws.top > 0 && c->s1_only != 1) {
          cudaEventRecord(c->ev_fork, s);
          cudaStreamWaitEvent(c->side, c->ev_fork, 0);
          if (c->h2d_on) cudaStreamWaitEvent(c->side, c->ev_h2d, 0);   // (overlapped upload: X^_1 present)
          kxk_lu_kernel<<<1, KXK_THREADS, std::max(c->k <= 64 ? 4 * c->k * c->k : c->k * c->k, PANEL_SMEM) * 8,
                          c->side>>>(ws, X);
          cudaEventRecord(c->ev_join, c->side);
          ++n;
        }
        // S1: W = A X - shift X, or (opts.square, Sec. 5.2) T = A X into X~'s buffer, then
        // W = A T - shift X; the alpha / g partials are those of the last product.
        // (world > 1: T's rows from the other ranks are exchanged between the products, s1_only)
        const int npass = c->opts.square ? 2 : 1;
        const int pass0 = c->s1_only == 1 ? 1 : 0, pass1 = c->s1_only == 0 ? 1 : npass;
        for (int pass = pass0; pass < pass1; ++pass) {
          const bool last = pass + 1 == npass;
          Ws wp = ws;
          if (!last) wp.shift = 0.0;
          const double* Xg = pass ? ws.Xt : X;                   // operand of this product
          if (!c->csr && c->oz_ns > 0) {   // A X on the INT8 tensor cores (ozaki.cuh)
            const double* Xb = c->multi ? c->Xfull : Xg;           // B operand: all n rows
            double* out = (c->oz_ns == 1) ? ws.W : ws.Wpart;
            if (pass == 0) c->mark();
            cudaMemsetAsync(c->oz_f, 0x80, c->k * sizeof(int32_t), s);
            oz_colexp_kernel<<<c->sms * 4, 256, 0, s>>>(Xb, c->n, c->k, c->oz_f);
            oz_slice_X_kernel<<<c->sms * 8, 256, 0, s>>>(Xb, c->n, c->k, c->oz_f, c->oz_X, c->oz_nks);
            const dim3 g((unsigned)c->oz_nrt, (unsigned)c->oz_ns);
            switch (c->k) {
              case 16: oz_gemm_kernel<16><<<g, OZ_THREADS, OzCfg<16>::SMEM, s>>>(c->oz_A, c->oz_X, c->oz_e, c->oz_f, c->n_loc, c->oz_nks, c->oz_ks_per, out, c->n_loc * c->k, c->oz_diag, Xb, c->row_begin, ws.status); break;
              case 32: oz_gemm_kernel<32><<<g, OZ_THREADS, OzCfg<32>::SMEM, s>>>(c->oz_A, c->oz_X, c->oz_e, c->oz_f, c->n_loc, c->oz_nks, c->oz_ks_per, out, c->n_loc * c->k, c->oz_diag, Xb, c->row_begin, ws.status); break;
              case 48: oz_gemm_kernel<48><<<g, OZ_THREADS, OzCfg<48>::SMEM, s>>>(c->oz_A, c->oz_X, c->oz_e, c->oz_f, c->n_loc, c->oz_nks, c->oz_ks_per, out, c->n_loc * c->k, c->oz_diag, Xb, c->row_begin, ws.status); break;
              default: oz_gemm_kernel<64><<<g, OZ_THREADS, OzCfg<64>::SMEM, s>>>(c->oz_A, c->oz_X, c->oz_e, c->oz_f, c->n_loc, c->oz_nks, c->oz_ks_per, out, c->n_loc * c->k, c->oz_diag, Xb, c->row_begin, ws.status); break;
            }
            if (last) c->mark();
            w_finish_kernel<<<c->w_fin_grid, 256, 0, s>>>(wp, X, c->oz_ns, c->n_loc * c->k);
            c->n_ag_cur = c->w_fin_grid;
            n += 4;
          } else if (!c->csr) {
            const double* Xb = c->multi ? c->Xfull : Xg;           // B operand: all n rows
            const bool bv16 = xv16 && ((uintptr_t)Xb % 16 == 0);
            const bool av16 = (c->n % 2 == 0) && (c->lda % 2 == 0) && ((uintptr_t)c->A % 16 == 0) && (c->kchunk % 2 == 0);
            double* out = (c->nsplit == 1) ? ws.W : ws.Wpart;
            // split-K fix-up + shift + alpha/g partials in the GEMM's last CTA per row tile (fused_finish),
            // else by w_finish
            FusedFinish fin{wp, X, c->gemm_cnt, c->wfuse ? 1 : 0};
            if (pass == 0) c->mark();
            const bool tma = TMA_OK && c->gemm_tma && bv16 && gemm_x_map(c, Xb);
            const bool poll = c->h2d_on && tma && !c->multi && pass == 0;   // S1 consumes X^ as it arrives
            if (c->h2d_on && !poll) cudaStreamWaitEvent(s, c->ev_h2d, 0);
            if (poll) {
              fin.ready = c->h2d_ready;
              fin.epoch = c->h2d_epoch;
              fin.ready_rows = c->h2d_rows;
            }
            if (tma)
              launch_k(c->pdl, gemm_tma, dim3(c->nsplit, c->gemm_gx), dim3(TGC::THREADS + 32), T_SMEM, s,
                       c->tm_A, c->tm_X, c->k, c->n_loc, c->n, c->kchunk, out, c->n_loc * c->k, ws.status, fin);
            else
              launch_k(c->pdl, gemm, dim3(c->nsplit, c->gemm_gx), dim3(GC::THREADS), GC::SMEM, s, c->A, c->lda, Xb,
                       c->k, c->n_loc, c->n, c->kchunk, out, c->n_loc * c->k, av16, bv16, ws.status, fin);
            if (last) c->mark();
            if (poll) cudaStreamWaitEvent(s, c->ev_h2d, 0);   // everything after S1 sees all of X^
            if (c->wfuse) {
              c->n_ag_cur = c->gemm_gx;
              n += 1;
            } else {
              c->n_ag_cur = c->w_fin_grid;
              launch_k(c->pdl, w_finish_kernel, dim3(c->w_fin_grid), dim3(256), 0, s, wp, (const double*)X, c->nsplit,
                       c->n_loc * c->k);
              n += 2;
            }
          } else {
            if (pass == 0) c->mark();
            const bool vec = xv16 && (c->k & (c->k - 1)) == 0 && c->k >= 2 &&
                             (ws.halo == nullptr || (uintptr_t)ws.halo % 16 == 0);
            if (ws.halo) launch_spmm<true>(c, vec, Xg, X, wp);
            else launch_spmm<false>(c, vec, Xg, X, wp);
            n += 1;
          }
          if (!last) cudaMemcpyAsync(ws.Xt, ws.W, (size_t)c->n_loc * c->k * 8, cudaMemcpyDeviceToDevice, s);   // T = A X
        }
        if (ph == 0 && c->multi && pass1 == npass) {
          ws.n_ag = c->n_ag_cur;
          ag_local_kernel<<<1, KXK_THREADS, 0, s>>>(ws);
          ++n;
        }
        break;
      }
      case 11: {  // Rayleigh-Ritz: pass B with D = 0 -> M2 = X_2^T W_2, G2 = X_2^T X_2
        Ws wz = ws;
        wz.d = ws.zerod;
        if (B2 && B2C::PAIRED)
          passB<<<dim3(7 * (c->passb_grid_y / 2)), B_THREADS, B_SMEM, s>>>(wz, X, xv16);
        else
          passB<<<dim3(B_NT, c->passb_grid_y), B_THREADS, B_SMEM, s>>>(wz, X, xv16);
        passBred<<<(2 * c->k * c->k + c->k + 31) / 32, PB_RED_THREADS, 0, s>>>(ws, c->passb_grid_y);
        n += 2;
        break;
      }
      case 12:  // Rayleigh-Ritz k x k stage (rank 0)
      case 13:  // reorthogonalisation (Cholesky QR) k x k stage (rank 0)
        if (c->rank == 0) {
          rr_kxk_kernel<<<1, KXK_THREADS, PANEL_SMEM * 8, s>>>(ws, X, ws.W, ph == 13 ? 1 : 0);
          n += 1;
        }
        break;
      case 1:  // S2: alpha, Rayleigh quotients
        c->mark();
        ws.n_ag = c->n_ag_cur;   // slots of the S1 kernel that ran (gather or stencil SpMM)
        launch_k(c->pdl, kxk_rq_kernel, dim3(1), dim3(KXK_THREADS), 0, s, ws);
        n += 1;
        break;
      case 2:  // S4 reductions
        c->mark();
        if (use_tc(c, X)) {   // NEXT-2: X_2^T [R_2 | X_2] on tcgen05, one FP64 partial per SM
          Ws wb = ws;
          wb.bdiag = c->bdiag;   // + the FP64 diagonals of M2, G2
          passB_tc_kernel<TKP><<<c->sms, TCB_THREADS, TcbCfg<TKP>::SMEM, s>>>(wb, X);
          c->mark();
          passB2_reduce_kernel<(KP >= 32 ? KP : 32)><<<(2 * c->k * c->k + c->k + 31) / 32, PB_RED_THREADS, 0, s>>>(
              wb, c->sms);
          n += 2;
          break;
        }
        if (B2 && B2C::PAIRED && c->pb_tma && c->pb_pp && xv16 && passb_x_map(c, X))
          launch_k(c->pdl, passB2_pp_kernel, dim3(7 * (c->passb_grid_y / 2)), dim3(PassB2PPCfg::THREADS),
                   PassB2PPCfg::SMEM, s, ws, c->tm_Xb, c->tm_Wb);
        else if (B2 && B2C::PAIRED && c->pb_tma && xv16 && passb_x_map(c, X))
          launch_k(c->pdl, passB2_tma_kernel<128>, dim3(7 * (c->passb_grid_y / 2)), dim3(PassB2TmaCfg<128>::THREADS + 32),
                   PassB2TmaCfg<128>::SMEM, s, ws, c->tm_Xb, c->tm_Wb);
        else if (B2 && B2C::PAIRED)
          launch_k(c->pdl, passB, dim3(7 * (c->passb_grid_y / 2)), dim3(B_THREADS), B_SMEM, s, ws, (const double*)X,
                   (int)xv16);
        else
          launch_k(c->pdl, passB, dim3(B_NT, c->passb_grid_y), dim3(B_THREADS), B_SMEM, s, ws, (const double*)X,
                   (int)xv16);
        c->mark();
        launch_k(c->pdl, passBred, dim3((2 * c->k * c->k + c->k + 31) / 32), dim3(PB_RED_THREADS), 0, s, ws,
                 c->passb_grid_y);
        n += 2;
        break;
      case 3:  // k x k algebra (rank 0), after the side-stream S3 joins
        c->mark();
        if (c->rank == 0) {
          cudaStreamWaitEvent(s, c->ev_join, 0);
          const cudaError_t e = launch_kxk_finish(ws, X, s, c->pdl);
          if (e != cudaSuccess) {   // (sticky: enqueue_phases reports it through the context)
            cuda_fail(c, e, "kxk_finish launch");
            return n;
          }
          n += 1;
        }
        break;
      case 4:  // S6 (+ S7: a sweep's Csig / scal already carry 1 / ||x~_j||, so pass C writes the
               // final X in place; Rayleigh-Ritz / QR steps write X~ and normalise in phase 5)
        c->mark();
        if (!c->in_rr) {
          if (KP == 128 && c->opts.emul && c->k == 128 && ((uintptr_t)X % 16 == 0))   // X_2 Csig on INT8
            passC_oz_kernel<<<c->sms, OZC_THREADS, OZC_SMEM, s>>>(ws, X, X);
          else if (use_tc_c(c, X))   // NEXT-2: X_2 Csig on tcgen05
            passC_tc_kernel<TKP><<<c->sms, TCC_THREADS, TccCfg<TKP>::SMEM, s>>>(ws, X, X);
          else if (KP == 128 && c->pc_pp == 4 && xv16 && passc3_x_map(c, X, PassCPP4Cfg::BR))   // 4 stages of 16 rows
            launch_k(c->pdl, passC_pp_kernel<PassCPP4Cfg>, dim3(c->sms), dim3(PassCPP4Cfg::BLOCK), PassCPP4Cfg::SMEM, s,
                     ws, c->tm_Xc, X);
          else if (KP == 128 && c->pc_pp == 3 && xv16 && passc3_x_map(c, X, PassCPP3Cfg::BR))   // 3 stages of 24 rows
            launch_k(c->pdl, passC_pp_kernel<PassCPP3Cfg>, dim3(c->sms), dim3(PassCPP3Cfg::BLOCK), PassCPP3Cfg::SMEM, s,
                     ws, c->tm_Xc, X);
          else if (KP == 128 && c->pc_pp && xv16 && passb_x_map(c, X))   // ping-pong pass C (X's pass-B map)
            launch_k(c->pdl, passC_pp_kernel<PassCPPCfg>, dim3(c->sms), dim3(PassCPPCfg::BLOCK), PassCPPCfg::SMEM, s, ws,
                     c->tm_Xb, X);
          else
            launch_k(c->pdl, passC_sweep, dim3(c->passc_grid, 1), dim3(CC::THREADS), CC::SMEM, s, ws,
                     (const double*)X, X, (int)xv16);
          n += 1;
          break;
        }
        passC<<<dim3(c->passc_grid, 1), CC::THREADS, CC::SMEM, s>>>(ws, X, ws.Xt, xv16);
        c->mark();
        norm_reduce_kernel<<<1, KXK_THREADS, 0, s>>>(ws);
        n += 2;
        break;
      case 5:  // S7 (Rayleigh-Ritz / QR steps; a sweep normalised in kxk_finish / pass C)
        if (!c->in_rr) {
          c->mark();
          break;
        }
        if (c->opts.normalize) {
          c->mark();
          normalize_kernel<<<c->sms * 8, 256, 0, s>>>(ws, X);
          ++n;
        } else {
          copy_gated_kernel<<<c->sms * 4, 256, 0, s>>>(ws.status, X, ws.Xt, c->n_loc * c->k);
          ++n;
        }
        c->mark();
        break;
    }
    return n;
  }
};

template <typename F>
static auto dispatch(int kp, F&& f) {
  switch (kp) {
    case 8: return f(Kern<8>{});
    case 16: return f(Kern<16>{});
    case 32: return f(Kern<32>{});
    case 64: return f(Kern<64>{});
    default: return f(Kern<128>{});
  }
}

// ---------------------------------------------------------------- init
static refine_ctx* ctx0(refine_ctx* c) { return c->loopback ? c->kids[0] : c; }

// spmm_gather_kernel eligibility and geometry (k a power of two <= 128, 32-bit gather offsets):
// resident grid and the largest rows-per-chunk R whose chunks all fit the staged nonzero buffer.
template <int K, int UN>
static cudaError_t gather_geometry_un(refine_ctx* c, const std::vector<int32_t>& rp) {
  using G = GatherCfg<K, UN>;
  int occ = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, spmm_gather_kernel<K, false, UN>, 256, 0);
  if (e != cudaSuccess) return e;
  int occ2 = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ2, spmm_gather_kernel<K, true, UN>, 256, 0);
  if (e != cudaSuccess) return e;
  occ = std::max(1, std::min(occ, occ2));
  const int64_t n = c->n_loc;
  int R = 0;
  for (int r = G::RMAX; r >= 1 && R == 0; r = (r > G::RG) ? r - G::RG : r / 2) {
    int64_t worst = 0;
    for (int64_t i = 0; i < n; i += r) worst = std::max<int64_t>(worst, (int64_t)rp[std::min<int64_t>(i + r, n)] - rp[i]);
    if (worst <= G::NZCAP) R = r;
  }
  c->gather_R = R;
  c->gather_un = UN;
  if (R > 0) {
    const int64_t chunks = (n + R - 1) / R;
    // rank 0 leaves one SM to kxk_lu (one 1024-thread CTA forked onto the side stream): a
    // persistent grid sized to every SM would otherwise park one SM's CTAs behind it
    const int sms = (c->rank == 0 && c->sms > 1) ? c->sms - 1 : c->sms;
    c->spmm_grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)sms * occ, chunks));
  }
  return cudaSuccess;
}

static cudaError_t gather_order(refine_ctx* c, const std::vector<int32_t>& rp, int RG, int nzcap);

// batch size UN: the smallest of {5, 7, 8} covering 95% of the rows (the stencils' 5 / 7)
template <int K>
static cudaError_t gather_geometry(refine_ctx* c, const std::vector<int32_t>& rp) {
  const int64_t n = c->n_loc;
  int64_t cnt[10] = {0};
  for (int64_t i = 0; i < n; ++i) cnt[std::min<int64_t>(rp[i + 1] - rp[i], 9)]++;
  int64_t acc = 0;
  int p95 = 9;
  for (int v = 0; v <= 9; ++v) {
    acc += cnt[v];
    if (acc * 100 >= n * 95) { p95 = v; break; }
  }
  cudaError_t e;
  if (p95 <= 5) e = gather_geometry_un<K, 5>(c, rp);
  else if (p95 <= 7) e = gather_geometry_un<K, 7>(c, rp);
  else e = gather_geometry_un<K, 8>(c, rp);
  if (e != cudaSuccess) return e;
  return gather_order(c, rp, GatherCfg<K>::RG, GatherCfg<K>::NZCAP);
}

// Stencil-aware chunk order for the gather kernel (spmm_csr.cuh chunk_of): the row offsets present
// in (nearly) every sampled row; three levels {1, d2, d3} with d2 | d3 (a 3-D stencil in
// lexicographic order) and a +-d3 reuse window larger than about a fifth of L2 select the tiled
// order; the chunk size becomes the largest divisor of d2 not above R and not below the row groups.
// REFINE_SPMM_ORDER=1 forces it whenever the structure is found (tests), =0 disables it.
static cudaError_t gather_order(refine_ctx* c, const std::vector<int32_t>& rp, int RG, int nzcap) {
  c->spmm_ord = make_int4(0, 0, 0, 0);
  const char* env = getenv("REFINE_SPMM_ORDER");
  if ((env && env[0] == '0') || c->multi || c->gather_R <= 0) return cudaSuccess;
  const int64_t S = std::min<int64_t>(c->n_loc, 65536);
  const int64_t nz = (int64_t)rp[S] - rp[0];
  if (S < 64 || nz <= 0) return cudaSuccess;
  std::vector<int32_t> ci(nz);
  cudaError_t e = cudaMemcpy(ci.data(), c->ci + rp[0], nz * sizeof(int32_t), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return e;
  std::vector<std::pair<int64_t, int64_t>> cnt;          // (offset, count), few distinct offsets
  for (int64_t i = 0; i < S; ++i)
    for (int32_t q = rp[i]; q < rp[i + 1]; ++q) {
      const int64_t o = std::llabs((int64_t)ci[q - rp[0]] - (c->row_begin + i));
      if (o == 0) continue;
      auto it = std::find_if(cnt.begin(), cnt.end(), [&](const std::pair<int64_t, int64_t>& p) { return p.first == o; });
      if (it != cnt.end()) ++it->second;
      else if (cnt.size() < 16) cnt.push_back({o, 1});
      else return cudaSuccess;                              // not a stencil
    }
  std::vector<int64_t> lv;
  for (auto& p : cnt)
    if (p.second >= S / 4) lv.push_back(p.first);
  std::sort(lv.begin(), lv.end());
  if (lv.size() != 3 || lv[0] != 1 || lv[2] % lv[1] != 0) return cudaSuccess;
  const int64_t d2 = lv[1], d3 = lv[2];
  const bool force = env && env[0] == '1';
  if (!force && 2 * d3 * c->k * 8 < (int64_t)24 << 20) return cudaSuccess;   // window fits L2 already
  int R = 0;
  for (int r = std::min<int>(c->gather_R, (int)d2); r >= RG; --r)
    if (d2 % r == 0) { R = r; break; }                  // (r >= RG: every row group busy)
  if (R == 0) return cudaSuccess;
  // the new chunks [q R, (q + 1) R) must each fit the staged nonzero buffer over ALL rows (the
  // stencil test above only sampled the first rows); otherwise keep the identity order and old R
  for (int64_t i = 0; i < c->n_loc; i += R)
    if ((int64_t)rp[std::min<int64_t>(i + R, c->n_loc)] - rp[i] > nzcap) return cudaSuccess;
  c->gather_R = R;
  c->spmm_ord = make_int4((int)(d2 / R), (int)(d3 / d2), 16, (int)((c->n_loc + d3 - 1) / d3));   // 16 lines per tile
  return cudaSuccess;
}

static cudaError_t gather_setup(refine_ctx* c) {
  c->gather_R = 0;
  const int k = c->k;
  if (getenv("REFINE_NO_GATHER") || (k & (k - 1)) != 0 || k < 2 || k > 128) return cudaSuccess;
  if ((int64_t)(c->n - 0) * (k / 2) >= (int64_t(1) << 31)) return cudaSuccess;   // local + halo offsets in int32
  std::vector<int32_t> rp(c->n_loc + 1);
  cudaError_t e = cudaMemcpy(rp.data(), c->rp, rp.size() * sizeof(int32_t), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return e;
  switch (k) {
    case 2: return gather_geometry<2>(c, rp);
    case 4: return gather_geometry<4>(c, rp);
    case 8: return gather_geometry<8>(c, rp);
    case 16: return gather_geometry<16>(c, rp);
    case 32: return gather_geometry<32>(c, rp);
    case 64: return gather_geometry<64>(c, rp);
    default: return gather_geometry<128>(c, rp);
  }
}

// gather offsets of the local nonzeros (after the halo layout is known)
static cudaError_t gather_offsets(refine_ctx* c) {
  if (c->gather_R <= 0) return cudaSuccess;
  int32_t p[2];
  cudaError_t e = cudaMemcpy(&p[0], c->rp, sizeof(int32_t), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(&p[1], c->rp + c->n_loc, sizeof(int32_t), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return e;
  const int64_t nnz = (int64_t)p[1] - p[0];
  if ((e = cudaMalloc(&c->xoff_buf, std::max<int64_t>(nnz, 1) * sizeof(int32_t))) != cudaSuccess) return e;
  c->xoff = c->xoff_buf - p[0];                    // indexed by absolute CSR position, like col_idx
  if (nnz > 0)
    spmm_xoff_kernel<<<c->sms * 8, 256, 0, c->stream>>>(c->ci + p[0], nnz, c->ws.row0, c->ws.row1,
                                                        c->ws.halo ? c->ws.halo_lo : c->ws.row0, c->k / 2,
                                                        c->xoff_buf);
  return cudaGetLastError();
}

// Per-rank setup: launch geometry, workspace pool, local ||A - shift I||_inf row maxima and (CSR)
// the range of referenced columns.  Cross-rank quantities are settled by finalize_partition.
static refine_status init_rank(refine_ctx* c, int64_t n, int32_t k, int64_t row_begin, int64_t row_end,
                               double shift, int rank, int world, const refine_opts* opts, void* stream,
                               double* local_norm, int64_t* col_lo, int64_t* col_hi) {
  if (k < 1 || (int64_t)k >= n || row_begin < 0 || row_end > n || row_end <= row_begin) return REFINE_E_INVALID;
  if (k > KMAX) return REFINE_E_UNSUPPORTED;
  c->rank = rank;
  c->world = world;
  if (c->rank == 0 && (row_begin != 0 || row_end - row_begin < k)) return REFINE_E_INVALID;
  c->n = n; c->k = k; c->kp = pad_kp(k);
  c->row_begin = row_begin; c->row_end = row_end; c->n_loc = row_end - row_begin;
  c->shift = shift;
  c->opts = refine_opts{10.0, 0, 1, 3, 10.0, 0, 0, 0.0, 0.0, 0, 0, 0};
  if (opts) c->opts = *opts;
  c->stream = (cudaStream_t)stream;
  RF_CK(c, cudaGetDevice(&c->device));
  RF_CK(c, cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, c->device));
  Ws& ws = c->ws;
  ws.n_loc = c->n_loc; ws.k = k; ws.kp = c->kp;
  ws.top = (c->rank == 0) ? k : 0;
  ws.shift = shift;
  ws.beta_zero = c->opts.beta_zero;
  ws.kjudge = c->opts.kjudge;
  // the divergence guard compares with the corr norm guard_window sweeps back (a 4-entry ring)
  if (c->opts.guard_window < 0 || c->opts.guard_window > 4) return REFINE_E_INVALID;
  if (c->opts.mixed && (k % 16 != 0 || k < 32)) return REFINE_E_UNSUPPORTED;    // tcgen05 passes: 16 | k >= 32
  // ozaki.cuh: dense S1 for 16 | k <= 64, pass C for k == 128 -- at least one must apply
  const bool emul_s1 = c->opts.emul && !c->csr && k % 16 == 0 && k <= 64;
  if (c->opts.emul && !emul_s1 && k != 128) return REFINE_E_UNSUPPORTED;
  if (emul_s1) {   // split the K range so each CTA's int32 levels stay exact, waves near-full
    c->oz_nks = (c->n + OZ_BK - 1) / OZ_BK;
    c->oz_nrt = (c->n_loc + OZ_BM - 1) / OZ_BM;
    const int64_t ns_min = (c->oz_nks + (OZ_KMAX / OZ_BK) - 1) / (OZ_KMAX / OZ_BK);
    int best = (int)ns_min;
    double best_eff = -1.0;
    for (int64_t ns = ns_min; ns <= std::max<int64_t>(ns_min, 16); ++ns) {
      const int64_t ctas = c->oz_nrt * ns;
      const double eff = (double)ctas / ((double)((ctas + c->sms - 1) / c->sms) * c->sms);
      if (eff > best_eff + 0.01) { best_eff = eff; best = (int)ns; }
    }
    c->oz_ks_per = (c->oz_nks + best - 1) / best;
    c->oz_ns = (int)((c->oz_nks + c->oz_ks_per - 1) / c->oz_ks_per);
  }
  ws.world = world; ws.rank = rank;
  ws.multi = c->multi ? 1 : 0;
  ws.row0 = row_begin; ws.row1 = row_end;
  ws.halo = nullptr; ws.halo_lo = row_begin;
  {
    const char* pe = getenv("REFINE_PDL");
    c->pdl = !(pe && pe[0] == '0');
  }
  if (!c->csr) {   // TMA-fed S1: A row stride and base 16-byte aligned, k even; REFINE_GEMM_TMA=0 disables
    const char* ge = getenv("REFINE_GEMM_TMA");
    c->gemm_tma = !(ge && ge[0] == '0') && k % 2 == 0 && c->kp >= 16 &&
                  encode_2d(&c->tm_A, c->A, (uint64_t)n, (uint64_t)c->n_loc, (uint64_t)c->lda,
                            (uint32_t)dispatch(c->kp, [&](auto K) { return decltype(K)::GBM; }));
  }
  if (c->kp == 128) {   // TMA-fed pass B at k = 128 (REFINE_PASSB_TMA=0 disables)
    const char* pe = getenv("REFINE_PASSB_TMA");
    c->pb_tma = !(pe && pe[0] == '0') && k % 2 == 0 && tensor_map_encoder() != nullptr;
    if (c->pb_tma)
      RF_CK(c, cudaFuncSetAttribute(passB2_tma_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    PassB2TmaCfg<128>::SMEM));
    // the ping-pong pass B (passB2_pp_kernel; REFINE_PASSB_PP=0 keeps passB2_tma_kernel)
    const char* bpe = getenv("REFINE_PASSB_PP");
    c->pb_pp = c->pb_tma && !(bpe && bpe[0] == '0');
    if (c->pb_pp)
      RF_CK(c, cudaFuncSetAttribute(passB2_pp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, PassB2PPCfg::SMEM));
    // k = 128 (even): the ping-pong pass C (passC_pp_kernel; REFINE_PASSC_PP=0 disables): 3 stages of 24
    // rows by default (cfg5 4.00 ms), 1: 2 stages of 32 rows (4.15 ms), 4: 4 stages of 16 rows (4.01 ms)
    const char* ce = getenv("REFINE_PASSC_PP");
    c->pc_pp = (!(ce && ce[0] == '0') && c->k == 128 && tensor_map_encoder() != nullptr) ? ((ce && (ce[0] == '1' || ce[0] == '4')) ? ce[0] - '0' : 3) : 0;
    if (c->pc_pp) {
      RF_CK(c, cudaFuncSetAttribute(passC_pp_kernel<PassCPPCfg>, cudaFuncAttributeMaxDynamicSharedMemorySize, PassCPPCfg::SMEM));
      RF_CK(c, cudaFuncSetAttribute(passC_pp_kernel<PassCPP3Cfg>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    PassCPP3Cfg::SMEM));
      RF_CK(c, cudaFuncSetAttribute(passC_pp_kernel<PassCPP4Cfg>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    PassCPP4Cfg::SMEM));
    }
  }
  RF_CK(c, (cudaError_t)dispatch(c->kp, [&](auto K) { return decltype(K)::setup(c); }));
  RF_CK(c, cudaFuncSetAttribute(kxk_lu_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, std::max(KMAX * KMAX, std::max(PANEL_SMEM, 4 * 64 * 64)) * 8));
  RF_CK(c, cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
  RF_CK(c, cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
  RF_CK(c, cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
  RF_CK(c, cudaFuncSetAttribute(kxk_finish_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, FK_SMEM * 8));
  RF_CK(c, cudaFuncSetAttribute(kxk_finish_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                kxk_small_smem_doubles(KXK_SMALL) * 8));
  RF_CK(c, cudaFuncSetAttribute(rr_kxk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, PANEL_SMEM * 8));
  // workspace sizes (doubles)
  size_t bpart = 0, brr = 0, nslot = 0;
  dispatch(c->kp, [&](auto K) { decltype(K)::sizes(c, bpart, brr, nslot); return 0; });
  // w_finish blocks = alpha/g slots that kxk_rq reduces on one SM: 4 per SM where w_finish streams
  // a large W (cfg3: 2 per SM doubles its time), 2 per SM below (cfg2: kxk_rq 15.8 -> 12.2 us)
  const int wf_per_sm = getenv("REFINE_WF_PER_SM") ? atoi(getenv("REFINE_WF_PER_SM")) : ((c->n_loc * (int64_t)k >= (int64_t)1 << 20) ? 4 : 2);
  c->w_fin_grid = (int)std::max<int64_t>(1, std::min<int64_t>(c->sms * wf_per_sm, c->n_loc / 2));
  c->spmm_grid = (int)std::max<int64_t>(1, std::min<int64_t>(c->sms * 8, (c->n_loc + 7) / 8));
  if (c->csr) RF_CK(c, gather_setup(c));
  if (c->csr) RF_CK(c, stencil_setup(c));
  // fused split-K fix-up: the last CTA of a row tile reads its nsplit partials, so only for a few splits
  // (measured: cfg1 (4 splits) 43.9 -> 43.0 us, cfg3 (4) 4.28 -> 4.27 ms, cfg2 (28 splits) 78 -> 84 us)
  const char* wf = getenv("REFINE_WFUSE");
  c->wfuse = !c->csr && c->oz_ns == 0 && (wf ? wf[0] != '0' : c->nsplit <= 8);
  c->n_ag = c->csr ? std::max(c->spmm_grid, c->st_on ? c->st_grid / c->st_geo.nq : 0)
                   : std::max(c->w_fin_grid, c->wfuse ? c->gemm_gx : 0);
  c->n_ag_cur = c->n_ag;
  const size_t nk = (size_t)c->n_loc * k, kk = (size_t)k * k, P = (size_t)world;
  const int nsplit_max = std::max(c->nsplit, c->oz_ns);
  const size_t wpart = (!c->csr && nsplit_max > 1) ? (size_t)nsplit_max * nk : 0;
  c->bc_cnt = kk + k + 8 + k + 1;   // [Csig | scal | stats(8) | ritz(k) | status]
  size_t off = 0;
  auto take = [&](size_t cnt) { size_t o = off; off += (cnt + 31) & ~size_t(31); return o; };
  const size_t oW = take(nk), oXt = take(nk), oWp = take(wpart), oAg = take((size_t)c->n_ag * k * 4), oBp = take(bpart),
               oBrr = take(brr), oMg = take(2 * kk + k), oNs = take(nslot),
               oAl = take(k), oD = take(k), oRd = take(k), oSg = take(k), oU = take(kk), oL = take(kk),
               oT = take(kk), oUi = take(kk), oE = take(kk), oBc = take(c->bc_cnt), oNt = take(k), oIn = take(k),
               oScr = take(KXK_SCRATCH_MATS * kk + KXK_SCRATCH_EXTRA), oRows = take((size_t)c->n_loc), oRun = take(8),
               oAgS = take(4 * k), oAgA = take(P * 4 * k), oMgA = take(c->multi ? P * (2 * kk + k) : 0),
               oNrS = take(k), oNrA = take(P * k), oCol = take(2), oZd = take(k), oGate = take(1),
               oBd = take(c->opts.mixed ? (size_t)c->sms * 2 * c->kp : 0), oCnt = take(c->wfuse ? (size_t)c->gemm_gx : 0);
  const size_t bytes = off * 8 + 64;
  RF_CK(c, cudaMalloc(&c->pool, bytes));
  c->pool_bytes = bytes;
  RF_CK(c, cudaMemsetAsync(c->pool, 0, bytes, c->stream));
  double* b = (double*)c->pool;
  ws.W = b + oW; ws.Xt = b + oXt;
  if (c->pb_tma)   // W's tensor map for the TMA-fed pass B (W lives in the pool)
    c->pb_tma = encode_2d(&c->tm_Wb, ws.W, (uint64_t)k, (uint64_t)c->n_loc, (uint64_t)k, PassB2TmaCfg<128>::BR); ws.Wpart = wpart ? b + oWp : nullptr; ws.ag = b + oAg; ws.n_ag = c->n_ag;
  ws.bpart = b + oBp; ws.brr = b + oBrr; ws.n_chunk = c->passb_grid_y;
  ws.M2 = b + oMg; ws.G2 = ws.M2 + kk; ws.rr2 = ws.M2 + 2 * kk;        // contiguous [M2 | G2 | rr2]
  ws.nslot = b + oNs; ws.n_nslot = c->passc_grid;
  ws.alpha = b + oAl; ws.d = b + oD; ws.rd = b + oRd; ws.sigma = b + oSg; ws.U = b + oU; ws.L = b + oL;
  ws.T = b + oT; ws.Uinv = b + oUi; ws.E11 = b + oE; ws.ntop = b + oNt; ws.invn = b + oIn;
  c->bc = b + oBc;                                   // [Csig | scal | stats(8) | ritz(k) | status]
  ws.Csig = c->bc; ws.scal = c->bc + kk; ws.stats = c->bc + kk + k;
  ws.ritz = c->bc + kk + k + 8;                      // (broadcast too: every rank reports the Ritz values)
  ws.status = reinterpret_cast<int*>(c->bc + kk + 2 * k + 8);
  ws.scratch = b + oScr;
  ws.ag_send = b + oAgS; ws.ag_all = b + oAgA; ws.mg_all = c->multi ? b + oMgA : nullptr;
  ws.nrm_send = b + oNrS; ws.nrm_all = b + oNrA;
  ws.zerod = b + oZd; ws.top_zero = 0;   // (the pool is zeroed below)
  c->gemm_cnt = c->wfuse ? reinterpret_cast<int*>(b + oCnt) : nullptr;   // (zeroed with the pool)
  ws.gate = reinterpret_cast<int*>(b + oGate);
  ws.want_gram = c->opts.reorth_tol > 0.0 ? 1 : 0;
  ws.normalize = c->opts.normalize ? 1 : 0;
  {   // the clustered kxk_finish (k > KXK_SMALL, or REFINE_KXK_SMALL=0) takes kxk_lu's H1..H4 (REFINE_KXK_H=0: off)
    const char* sm_ = getenv("REFINE_KXK_SMALL");
    const char* he = getenv("REFINE_KXK_H");
    ws.kxk_h = (!(he && he[0] == '0') && (k > KXK_SMALL || (sm_ && sm_[0] == '0'))) ? 1 : 0;
  }
  ws.bdiag = nullptr;
  ws.fk_nobulk = (getenv("REFINE_FK_BULK") && getenv("REFINE_FK_BULK")[0] == '0') ? 1 : 0;
  c->bdiag = c->opts.mixed ? b + oBd : nullptr;
  c->run = reinterpret_cast<RunState*>(b + oRun);
  ws.tlog = nullptr;
  if (getenv("REFINE_KXK_TIMING")) RF_CK(c, cudaMalloc(&ws.tlog, 64 * sizeof(long long)));
  // local rows of ||A - shift I||_inf (one pass over A) -> delta = c ||A|| u
  double* rows = b + oRows;
  const double nshift = c->opts.square ? 0.0 : shift;   // squared operator: ||A||_inf^2 + |shift| (SQ1)
  if (!c->csr)
    absrow_max_dense_kernel<<<c->sms * 8, 256, 0, c->stream>>>(c->A, c->lda, c->n_loc, c->n, c->row_begin, nshift, rows);
  else
    absrow_max_csr_kernel<<<c->sms * 8, 256, 0, c->stream>>>(c->rp, c->ci, c->val, c->n_loc, c->row_begin, nshift, rows);
  max_kernel<<<1, 1024, 0, c->stream>>>(rows, c->n_loc, ws.stats + 7);
  if (c->oz_ns > 0) {   // A's exponents and int8 slices, once (A is borrowed and constant)
    RF_CK(c, cudaMalloc(&c->oz_e, std::max<int64_t>(c->n_loc, 1) * sizeof(int32_t)));
    RF_CK(c, cudaMalloc(&c->oz_diag, std::max<int64_t>(c->n_loc, 1) * sizeof(double)));
    RF_CK(c, cudaMalloc(&c->oz_f, 64 * sizeof(int32_t)));
    RF_CK(c, cudaMalloc(&c->oz_A, (size_t)c->oz_nrt * c->oz_nks * OZ_S * OZ_ATILE));
    RF_CK(c, cudaMalloc(&c->oz_X, (size_t)c->oz_nks * OZ_S * k * OZ_BK));
    oz_rowexp_kernel<<<c->sms * 8, 256, 0, c->stream>>>(c->A, c->lda, c->n_loc, c->n, c->row_begin, c->oz_e, c->oz_diag);
    oz_slice_A_kernel<<<c->sms * 16, 256, 0, c->stream>>>(c->A, c->lda, c->n_loc, c->n, c->row_begin, c->oz_e, c->oz_A,
                                                          c->oz_nks);
    auto attr = [&](auto kern, int smem) { return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); };
    RF_CK(c, attr(oz_gemm_kernel<16>, OzCfg<16>::SMEM));
    RF_CK(c, attr(oz_gemm_kernel<32>, OzCfg<32>::SMEM));
    RF_CK(c, attr(oz_gemm_kernel<48>, OzCfg<48>::SMEM));
    RF_CK(c, attr(oz_gemm_kernel<64>, OzCfg<64>::SMEM));
  }
  unsigned long long* colr = reinterpret_cast<unsigned long long*>(b + oCol);
  if (c->csr && c->multi) {
    const unsigned long long init[2] = {~0ull, 0ull};
    RF_CK(c, cudaMemcpyAsync(colr, init, sizeof(init), cudaMemcpyHostToDevice, c->stream));
    col_range_kernel<<<c->sms * 4, 256, 0, c->stream>>>(c->rp, c->ci, c->n_loc, colr);
  }
  RF_CK(c, cudaGetLastError());
  unsigned long long cr[2] = {0, 0};
  RF_CK(c, cudaMemcpyAsync(local_norm, ws.stats + 7, 8, cudaMemcpyDeviceToHost, c->stream));
  if (c->csr && c->multi) RF_CK(c, cudaMemcpyAsync(cr, colr, sizeof(cr), cudaMemcpyDeviceToHost, c->stream));
  RF_CK(c, cudaStreamSynchronize(c->stream));
  *col_lo = (c->csr && c->multi) ? (int64_t)cr[0] : row_begin;
  *col_hi = (c->csr && c->multi) ? (int64_t)cr[1] : row_end - 1;
  if (*col_lo > row_begin) *col_lo = row_begin;
  if (*col_hi < row_end - 1) *col_hi = row_end - 1;
  return REFINE_OK;
}

// Halo plan of `rank` (see refine.h, refine_halo_plan): which X rows it receives from / sends to
// each other rank, with halo offsets (rows [lo, rb) first, then [re, hi]) and local offsets.
static void halo_plan(int world, int rank, const int64_t* rb, const int64_t* re, const int64_t* lo,
                      const int64_t* hi, std::vector<refine_ctx::Seg>& send, std::vector<refine_ctx::Seg>& recv,
                      int64_t* hrows) {
  send.clear();
  recv.clear();
  auto needs = [&](int r, int64_t out[4]) {
    out[0] = lo[r]; out[1] = rb[r];                       // [lo, rb)
    out[2] = re[r]; out[3] = hi[r] + 1;                   // [re, hi]
  };
  auto hidx = [&](int64_t g) { return g < rb[rank] ? g - lo[rank] : (rb[rank] - lo[rank]) + (g - re[rank]); };
  int64_t me[4];
  needs(rank, me);
  for (int s = 0; s < world; ++s) {
    if (s == rank) continue;
    for (int h = 0; h < 2; ++h) {                         // what I receive from s
      const int64_t a = std::max(me[2 * h], rb[s]), e = std::min(me[2 * h + 1], re[s]);
      if (e > a) recv.push_back({s, a, e - a, hidx(a)});
    }
    int64_t ns[4];
    needs(s, ns);
    for (int h = 0; h < 2; ++h) {                         // what s receives from me
      const int64_t a = std::max(ns[2 * h], rb[rank]), e = std::min(ns[2 * h + 1], re[rank]);
      if (e > a) send.push_back({s, a, e - a, a - rb[rank]});
    }
  }
  *hrows = std::max<int64_t>(rb[rank] - lo[rank], 0) + std::max<int64_t>(hi[rank] + 1 - re[rank], 0);
}

// Settle the cross-rank state of rank context c given every rank's rows, row maxima and column range.
static refine_status finalize_rank(refine_ctx* c, const std::vector<int64_t>& rb, const std::vector<int64_t>& re,
                                   const std::vector<double>& nrm, const std::vector<int64_t>& lo,
                                   const std::vector<int64_t>& hi) {
  const int P = c->world;
  if (rb[0] != 0 || re[P - 1] != c->n) return REFINE_E_INVALID;
  for (int r = 0; r + 1 < P; ++r)
    if (re[r] != rb[r + 1]) return REFINE_E_INVALID;       // ranks must tile [0, n) in rank order
  c->rb_all = rb;
  c->re_all = re;
  double normA = 0.0;
  for (double v : nrm) normA = std::max(normA, v);
  if (c->opts.square) normA = normA * normA + std::fabs(c->shift);   // bound of ||A^2 - shift I|| (SQ1)
  c->ws.normA = normA;
  c->ws.delta = c->opts.delta_c * normA * std::ldexp(1.0, -53);
  if (c->multi && c->csr) {
    int64_t hrows = 0;
    halo_plan(P, c->rank, rb.data(), re.data(), lo.data(), hi.data(), c->hsend, c->hrecv, &hrows);
    RF_CK(c, cudaMalloc(&c->ws.halo, std::max<int64_t>(hrows, 1) * c->k * sizeof(double)));
    c->ws.halo_lo = std::min(lo[c->rank], rb[c->rank]);
  }
  if (c->multi && !c->csr && !c->loopback_kid) {
    RF_CK(c, cudaMalloc(&c->Xfull, (size_t)c->n * c->k * sizeof(double)));
    c->own_xfull = true;
  }
  if (c->csr) RF_CK(c, gather_offsets(c));
  return REFINE_OK;
}

template <typename MakeRank>
static refine_status init_any(refine_ctx* c, int64_t n, int32_t k, int64_t row_begin, int64_t row_end, double shift,
                              const refine_comm* comm, const refine_opts* opts, void* stream, MakeRank make_rank) {
  const int world = comm ? comm->world : 1;
  const int rank = comm ? comm->rank : 0;
  if (world < 1 || rank < 0 || rank >= world) return REFINE_E_INVALID;
  if (world > 1 && comm->nccl_id == nullptr) {
    // loopback: `world` emulated ranks on this device, equal row blocks (rank 0 gets the rest)
    if (row_begin != 0 || row_end != n) return REFINE_E_INVALID;
    c->loopback = true;
    c->world = world;
    c->n = n; c->k = k; c->n_loc = n; c->row_begin = 0; c->row_end = n;
    c->stream = (cudaStream_t)stream;
    c->opts = refine_opts{10.0, 0, 1, 3, 10.0, 0, 0, 0.0, 0.0, 0, 0, 0};
    if (opts) c->opts = *opts;
    std::vector<int64_t> rb(world), re(world), lo(world), hi(world);
    std::vector<double> nrm(world);
    const int64_t blk = n / world;
    for (int r = 0; r < world; ++r) { rb[r] = r == 0 ? 0 : (n - blk * (world - r)); re[r] = n - blk * (world - r - 1); }
    c->multi = true;
    for (int r = 0; r < world; ++r) {
      refine_ctx* kid = new (std::nothrow) refine_ctx();
      if (!kid) return REFINE_E_NOMEM;
      c->kids.push_back(kid);
      kid->loopback_kid = true;
      kid->multi = true;
      make_rank(kid, rb[r]);
      refine_status st = init_rank(kid, n, k, rb[r], re[r], shift, r, world, opts, stream, &nrm[r], &lo[r], &hi[r]);
      if (st != REFINE_OK) return st;
    }
    for (auto* kid : c->kids) {
      refine_status st = finalize_rank(kid, rb, re, nrm, lo, hi);
      if (st != REFINE_OK) return st;
    }
    c->csr = c->kids[0]->csr;
    c->kp = c->kids[0]->kp;
    if (!c->csr && c->opts.square) RF_CK(c, cudaMalloc(&c->Tfull, (size_t)n * k * sizeof(double)));
    return REFINE_OK;
  }
  make_rank(c, row_begin);
  // NCCL path for world > 1; REFINE_FORCE_NCCL=1 also takes it at world == 1 (tests of the NCCL calls)
  c->multi = world > 1 || (comm && comm->nccl_id && getenv("REFINE_FORCE_NCCL"));
  double nrm = 0.0;
  int64_t lo = 0, hi = 0;
  refine_status st = init_rank(c, n, k, row_begin, row_end, shift, rank, world, opts, stream, &nrm, &lo, &hi);
  if (st != REFINE_OK) return st;
  if (!c->multi) {
    return finalize_rank(c, {row_begin}, {row_end}, {nrm}, {lo}, {hi});
  }
  // NCCL: one process per GPU; gather every rank's (rb, re, ||.||_inf rows, lo, hi)
  Nccl& N = nccl();
  if (!N.ok) return REFINE_E_NCCL;
  ncclUniqueId id;
  memcpy(&id, comm->nccl_id, sizeof(id));
  if (N.CommInitRank(&c->comm, world, id, rank) != ncclSuccess) return REFINE_E_NCCL;
  double* dv = nullptr;
  RF_CK(c, cudaMalloc(&dv, sizeof(double) * 5 * (world + 1)));
  const double mine[5] = {(double)row_begin, (double)row_end, nrm, (double)lo, (double)hi};
  RF_CK(c, cudaMemcpyAsync(dv, mine, sizeof(mine), cudaMemcpyHostToDevice, c->stream));
  if (N.AllGather(dv, dv + 5, 5, ncclDouble, c->comm, c->stream) != ncclSuccess) { cudaFree(dv); return REFINE_E_NCCL; }
  std::vector<double> all(5 * world);
  RF_CK(c, cudaMemcpyAsync(all.data(), dv + 5, sizeof(double) * 5 * world, cudaMemcpyDeviceToHost, c->stream));
  RF_CK(c, cudaStreamSynchronize(c->stream));
  cudaFree(dv);
  std::vector<int64_t> rb(world), re(world), lov(world), hiv(world);
  std::vector<double> nv(world);
  for (int r = 0; r < world; ++r) {
    rb[r] = (int64_t)all[5 * r]; re[r] = (int64_t)all[5 * r + 1]; nv[r] = all[5 * r + 2];
    lov[r] = (int64_t)all[5 * r + 3]; hiv[r] = (int64_t)all[5 * r + 4];
  }
  return finalize_rank(c, rb, re, nv, lov, hiv);
}

extern "C" refine_status refine_init_dense(refine_ctx** out, int64_t n, int32_t k, const double* A_rows, int64_t lda,
                                           int64_t row_begin, int64_t row_end, double shift,
                                           const refine_comm* comm, const refine_opts* opts, void* stream) {
  if (!out) return REFINE_E_INVALID;
  *out = nullptr;
  if (!A_rows || lda < n) return REFINE_E_INVALID;
  refine_ctx* c = new (std::nothrow) refine_ctx();
  if (!c) return REFINE_E_NOMEM;
  c->csr = false;
  refine_status st = init_any(c, n, k, row_begin, row_end, shift, comm, opts, stream, [&](refine_ctx* r, int64_t rb) {
    r->csr = false;
    r->lda = lda;
    r->A = (r == c || !c->loopback) ? A_rows : A_rows + rb * lda;   // loopback: rank r's row block
  });
  if (st != REFINE_OK) { refine_destroy(c); return st; }
  *out = c;
  return REFINE_OK;
}

extern "C" refine_status refine_init_csr(refine_ctx** out, int64_t n, int32_t k, const int32_t* row_ptr,
                                         const int32_t* col_idx, const double* val, int64_t row_begin,
                                         int64_t row_end, double shift, const refine_comm* comm,
                                         const refine_opts* opts, void* stream) {
  if (!out) return REFINE_E_INVALID;
  *out = nullptr;
  if (!row_ptr || !col_idx || !val) return REFINE_E_INVALID;
  refine_ctx* c = new (std::nothrow) refine_ctx();
  if (!c) return REFINE_E_NOMEM;
  c->csr = true;
  refine_status st = init_any(c, n, k, row_begin, row_end, shift, comm, opts, stream, [&](refine_ctx* r, int64_t rb) {
    r->csr = true;
    r->rp = (r == c || !c->loopback) ? row_ptr : row_ptr + rb;          // loopback: rank r's rows
    r->ci = col_idx;
    r->val = val;
  });
  if (st != REFINE_OK) { refine_destroy(c); return st; }
  *out = c;
  return REFINE_OK;
}

// ---------------------------------------------------------------- sweeps
enum { C_X = 0, C_AG, C_MG, C_BC, C_NRM, C_T };   // C_T: T = A X rows (opts.square)

static refine_status nccl_fail(refine_ctx* c, int r, const char* what) {
  Nccl& N = nccl();
  fprintf(stderr, "[refine] NCCL error in %s: %s\n", what, N.GetErrorString ? N.GetErrorString((ncclResult_t)r) : "?");
  c->sticky = REFINE_E_NCCL;
  return REFINE_E_NCCL;
}
#define RF_NC(c, expr)                                       \
  do {                                                       \
    int r_ = (int)(expr);                                    \
    if (r_ != 0) return nccl_fail((c), r_, #expr);           \
  } while (0)

// The cross-rank step `which` of one sweep.  c is the rank context (NCCL) or the loopback parent.
static refine_status collective(refine_ctx* c, int which, double* X) {
  const int64_t k = c->k;
  const cudaMemcpyKind D2D = cudaMemcpyDeviceToDevice;
  if (c->loopback) {
    auto& K = c->kids;
    const int P = (int)K.size();
    cudaStream_t s = c->stream;
    switch (which) {
      case C_X:
        for (auto* kid : K) {
          if (!kid->csr) { kid->Xfull = X; continue; }             // X already holds all n rows
          for (auto& g : kid->hrecv)
            RF_CK(c, cudaMemcpyAsync(kid->ws.halo + g.off * k, X + g.row * k, g.cnt * k * 8, D2D, s));
        }
        break;
      case C_AG:
        for (auto* kid : K)
          for (int r = 0; r < P; ++r)
            RF_CK(c, cudaMemcpyAsync(kid->ws.ag_all + r * 4 * k, K[r]->ws.ag_send, 4 * k * 8, D2D, s));
        break;
      case C_MG: {
        const int64_t cnt = 2 * k * k + k;
        for (int r = 0; r < P; ++r)
          RF_CK(c, cudaMemcpyAsync(K[0]->ws.mg_all + r * cnt, K[r]->ws.M2, cnt * 8, D2D, s));
        break;
      }
      case C_BC:
        for (int r = 1; r < P; ++r) RF_CK(c, cudaMemcpyAsync(K[r]->bc, K[0]->bc, K[0]->bc_cnt * 8, D2D, s));
        break;
      case C_NRM:
        for (auto* kid : K)
          for (int r = 0; r < P; ++r)
            RF_CK(c, cudaMemcpyAsync(kid->ws.nrm_all + r * k, K[r]->ws.nrm_send, k * 8, D2D, s));
        break;
      case C_T:   // every rank's T (its ws.Xt block): dense -> one full copy, CSR -> each rank's halo rows
        if (!c->csr) {
          for (auto* kid : K) RF_CK(c, cudaMemcpyAsync(c->Tfull + kid->row_begin * k, kid->ws.Xt, kid->n_loc * k * 8, D2D, s));
          for (auto* kid : K) kid->Xfull = c->Tfull;
        } else {
          for (auto* kid : K)
            for (auto& g : kid->hrecv) {
              const refine_ctx* o = K[g.peer];
              RF_CK(c, cudaMemcpyAsync(kid->ws.halo + g.off * k, o->ws.Xt + (g.row - o->row_begin) * k, g.cnt * k * 8, D2D, s));
            }
        }
        break;
    }
    return REFINE_OK;
  }
  Nccl& N = nccl();
  cudaStream_t s = c->stream;
  switch (which) {
    case C_X:
      RF_NC(c, N.GroupStart());
      if (!c->csr) {              // dense: every rank's block of X into the full copy
        for (int r = 0; r < c->world; ++r) {
          double* dst = c->Xfull + c->rb_all[r] * k;
          RF_NC(c, N.Broadcast(r == c->rank ? X : dst, dst, (c->re_all[r] - c->rb_all[r]) * k, ncclDouble, r,
                               c->comm, s));
        }
      } else {                    // CSR: halo rows only
        for (auto& g : c->hsend) RF_NC(c, N.Send(X + g.off * k, g.cnt * k, ncclDouble, g.peer, c->comm, s));
        for (auto& g : c->hrecv) RF_NC(c, N.Recv(c->ws.halo + g.off * k, g.cnt * k, ncclDouble, g.peer, c->comm, s));
      }
      RF_NC(c, N.GroupEnd());
      break;
    case C_AG:
      RF_NC(c, N.AllGather(c->ws.ag_send, c->ws.ag_all, 4 * k, ncclDouble, c->comm, s));
      break;
    case C_MG:
      RF_NC(c, N.AllGather(c->ws.M2, c->ws.mg_all, 2 * k * k + k, ncclDouble, c->comm, s));
      break;
    case C_BC:
      RF_NC(c, N.Broadcast(c->bc, c->bc, c->bc_cnt, ncclDouble, 0, c->comm, s));
      break;
    case C_NRM:
      RF_NC(c, N.AllGather(c->ws.nrm_send, c->ws.nrm_all, k, ncclDouble, c->comm, s));
      break;
    case C_T:   // as C_X, for T = A X (ws.Xt)
      RF_NC(c, N.GroupStart());
      if (!c->csr) {
        for (int r = 0; r < c->world; ++r) {
          double* dst = c->Xfull + c->rb_all[r] * k;
          RF_NC(c, N.Broadcast(r == c->rank ? c->ws.Xt : dst, dst, (c->re_all[r] - c->rb_all[r]) * k, ncclDouble, r,
                               c->comm, s));
        }
      } else {
        for (auto& g : c->hsend) RF_NC(c, N.Send(c->ws.Xt + g.off * k, g.cnt * k, ncclDouble, g.peer, c->comm, s));
        for (auto& g : c->hrecv) RF_NC(c, N.Recv(c->ws.halo + g.off * k, g.cnt * k, ncclDouble, g.peer, c->comm, s));
      }
      RF_NC(c, N.GroupEnd());
      break;
  }
  return REFINE_OK;
}

// One sweep's kernels and collectives (no status reset), every rank of c (loopback) or c itself.
static refine_status enqueue_phases(refine_ctx* c, double* X) {
  const bool multi = c->multi;
  refine_ctx* one[1] = {c};
  refine_ctx** ranks = c->loopback ? c->kids.data() : one;
  const int nr = c->loopback ? (int)c->kids.size() : 1;
  static const int after[6] = {C_AG, -1, C_MG, C_BC, -1, -1};
  refine_status st;
  if (multi && (st = collective(c, C_X, X)) != REFINE_OK) return st;
  int launches = 0;
  const bool split_s1 = multi && c->opts.square;   // T = A X, exchange T's rows, then W = A T - shift X
  for (int ph = 0; ph < 6; ++ph) {
    for (int part = 0; part < ((ph == 0 && split_s1) ? 2 : 1); ++part) {
      if (part == 1 && (st = collective(c, C_T, X)) != REFINE_OK) return st;
      for (int i = 0; i < nr; ++i) {
        refine_ctx* r = ranks[i];
        double* Xr = c->loopback ? X + r->row_begin * c->k : X;
        r->s1_only = (ph == 0 && split_s1) ? part : -1;
        launches += dispatch(r->kp, [&](auto K) { return decltype(K)::phase(r, ph, Xr); });
        r->s1_only = -1;
      }
    }
    if (multi && after[ph] >= 0 && (st = collective(c, after[ph], X)) != REFINE_OK) return st;
  }
  c->launches = launches;
  RF_CK(c, cudaGetLastError());
  for (int i = 0; i < nr; ++i)
    if (ranks[i]->sticky != REFINE_OK) return c->sticky = ranks[i]->sticky;
  return REFINE_OK;
}

static refine_status enqueue_sweep(refine_ctx* c, double* X) {
  if (c->loopback)
    for (auto* kid : c->kids) RF_CK(c, cudaMemsetAsync(kid->ws.status, 0, sizeof(int), c->stream));
  else
    RF_CK(c, cudaMemsetAsync(c->ws.status, 0, sizeof(int), c->stream));
  return enqueue_phases(c, X);
}

static refine_status launch_sweep(refine_ctx* c, double* X) {
  if (!c->use_graph) return enqueue_sweep(c, X);
  if (c->gexec == nullptr || c->gX != X) {
    if (c->gexec) { cudaGraphExecDestroy(c->gexec); c->gexec = nullptr; }
    cudaGraph_t g;
    if (!c->cap_stream) RF_CK(c, cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking));
    cudaStream_t user = c->stream;
    RF_CK(c, cudaStreamBeginCapture(c->cap_stream, cudaStreamCaptureModeThreadLocal));
    c->stream = c->cap_stream;
    for (auto* kid : c->kids) kid->stream = c->cap_stream;   // loopback: every emulated rank's launches
    refine_status st = enqueue_sweep(c, X);
    c->stream = user;
    for (auto* kid : c->kids) kid->stream = user;
    cudaError_t e = cudaStreamEndCapture(c->cap_stream, &g);
    if (st != REFINE_OK) return st;
    RF_CK(c, e);
    RF_CK(c, cudaGraphInstantiate(&c->gexec, g, 0));
    cudaGraphDestroy(g);
    c->gX = X;
  }
  RF_CK(c, cudaGraphLaunch(c->gexec, c->stream));
  return REFINE_OK;
}

// Rayleigh-Ritz preprocessing (Sec. 3.4): S1 -> pass B with D = 0 -> [gather]
// -> rr_kxk (rank 0) -> [broadcast Csig = -S, scal = 0] -> pass C (Z_2 = X_2 S) -> norms -> X = Z.
static refine_status enqueue_rr(refine_ctx* c, double* X, int mode = 0, bool gated = false) {
  // mode 0: Rayleigh-Ritz (S1, pass B with D = 0, rr_kxk, pass C, normalise);
  // mode 1: reorthogonalisation by Cholesky QR (pass B for G only, rr_kxk mode 1, pass C, normalise).
  // gated: refine_run's policy step -- every kernel runs behind ws.gate (no status reset).
  refine_ctx* one[1] = {c};
  refine_ctx** ranks = c->loopback ? c->kids.data() : one;
  const int nr = c->loopback ? (int)c->kids.size() : 1;
  if (!gated)
    for (int i = 0; i < nr; ++i) RF_CK(c, cudaMemsetAsync(ranks[i]->ws.status, 0, sizeof(int), c->stream));
  refine_status st;
  if (mode == 0 && c->multi && (st = collective(c, C_X, X)) != REFINE_OK) return st;
  static const int ph_rr[5] = {10, 11, 12, 4, 5}, ph_ro[5] = {11, 13, 4, 5, -1};
  static const int after[5] = {-1, C_MG, C_BC, C_NRM, -1}, after_ro[5] = {C_MG, C_BC, C_NRM, -1, -1};
  const int* phases = mode == 0 ? ph_rr : ph_ro;
  const int* aft = mode == 0 ? after : after_ro;
  const bool split_s1 = c->multi && c->opts.square;   // (as in enqueue_phases)
  for (int q = 0; q < 5 && phases[q] >= 0; ++q) {
    for (int part = 0; part < ((phases[q] == 10 && split_s1) ? 2 : 1); ++part) {
      if (part == 1 && (st = collective(c, C_T, X)) != REFINE_OK) return st;
      for (int i = 0; i < nr; ++i) {
        refine_ctx* r = ranks[i];
        double* Xr = c->loopback ? X + r->row_begin * c->k : X;
        r->gated = gated;
        r->in_rr = true;
        r->s1_only = (phases[q] == 10 && split_s1) ? part : -1;
        dispatch(r->kp, [&](auto K) { return decltype(K)::phase(r, phases[q], Xr); });
        r->gated = false;
        r->in_rr = false;
        r->s1_only = -1;
      }
    }
    if (c->multi && aft[q] >= 0 && (st = collective(c, aft[q], X)) != REFINE_OK) return st;
  }
  RF_CK(c, cudaGetLastError());
  return REFINE_OK;
}

static void set_top_zero(refine_ctx* c, int v) {
  if (c->loopback)
    for (auto* kid : c->kids) kid->ws.top_zero = v;
  c->ws.top_zero = v;
}

static refine_status map_status(int s) {
  switch (s) {
    case ST_OK: return REFINE_OK;
    case ST_DIVERGED: return REFINE_DIVERGED;
    case ST_E_INVALID: return REFINE_E_INVALID;
    case ST_E_NEAR_ZERO_RQ: return REFINE_E_NEAR_ZERO_RQ;
    case ST_E_ZERO_PIVOT: return REFINE_E_ZERO_PIVOT;
    default: return REFINE_E_CUDA;
  }
}

static refine_status read_stats(refine_ctx* c, refine_sweep_stats* stats, int* dev_status) {
  double h[8];
  int st = 0;
  const Ws& ws = ctx0(c)->ws;
  RF_CK(c, cudaMemcpyAsync(h, ws.stats, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
  RF_CK(c, cudaMemcpyAsync(&st, ws.status, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  RF_CK(c, cudaStreamSynchronize(c->stream));
  if (stats) {
    stats->rel_resid = h[0]; stats->corr_norm = h[1]; stats->min_gap = h[2];
    stats->delta_hits = (int32_t)h[3]; stats->flipped = (int32_t)h[4];
    stats->gram_dev = h[6];
  }
  *dev_status = st;
  return REFINE_OK;
}

extern "C" refine_status refine_rayleigh_ritz(refine_ctx* c, double* X, double* ritz) {
  if (!c || !X) return REFINE_E_INVALID;
  if (c->sticky != REFINE_OK) return c->sticky;
  refine_status st = enqueue_rr(c, X);
  if (st != REFINE_OK) return st;
  if (ritz) RF_CK(c, cudaMemcpyAsync(ritz, ctx0(c)->ws.ritz, sizeof(double) * c->k, cudaMemcpyDeviceToHost, c->stream));
  int dev = 0;
  RF_CK(c, cudaMemcpyAsync(&dev, ctx0(c)->ws.status, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  RF_CK(c, cudaStreamSynchronize(c->stream));
  return map_status(dev);
}

extern "C" refine_status refine_reorthogonalize(refine_ctx* c, double* X, double* gram_dev) {
  if (!c || !X) return REFINE_E_INVALID;
  if (c->sticky != REFINE_OK) return c->sticky;
  refine_status st = enqueue_rr(c, X, 1);
  if (st != REFINE_OK) return st;
  if (gram_dev) RF_CK(c, cudaMemcpyAsync(gram_dev, ctx0(c)->ws.ritz, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  int dev = 0;
  RF_CK(c, cudaMemcpyAsync(&dev, ctx0(c)->ws.status, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  RF_CK(c, cudaStreamSynchronize(c->stream));
  return map_status(dev);
}

extern "C" refine_status refine_sweep_rr(refine_ctx* c, double* X, refine_sweep_stats* stats, double* ritz) {
  if (!c || !X) return REFINE_E_INVALID;
  if (c->sticky != REFINE_OK) return c->sticky;
  refine_status st = enqueue_rr(c, X);
  if (st != REFINE_OK) return st;
  if (ritz) RF_CK(c, cudaMemcpyAsync(ritz, ctx0(c)->ws.ritz, sizeof(double) * c->k, cudaMemcpyDeviceToHost, c->stream));
  int dev = 0;
  RF_CK(c, cudaMemcpyAsync(&dev, ctx0(c)->ws.status, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  RF_CK(c, cudaStreamSynchronize(c->stream));
  if (dev != ST_OK) return map_status(dev);
  set_top_zero(c, 1);
  st = enqueue_sweep(c, X);          // direct launches (the cached sweep graph has top_zero = 0)
  set_top_zero(c, 0);
  if (st != REFINE_OK) return st;
  if ((st = read_stats(c, stats, &dev)) != REFINE_OK) return st;
  return map_status(dev);
}

extern "C" refine_status refine_sweep(refine_ctx* c, double* X, refine_sweep_stats* stats) {
  if (!c || !X) return REFINE_E_INVALID;
  if (c->sticky != REFINE_OK) return c->sticky;
  refine_status st = launch_sweep(c, X);
  if (st != REFINE_OK || !stats) return st;
  int ds = 0;
  if ((st = read_stats(c, stats, &ds)) != REFINE_OK) return st;
  return map_status(ds);
}

extern "C" refine_status refine_sweep_host(refine_ctx* c, const double* X_host_in, double* X_host_out,
                                           refine_sweep_stats* stats) {
  if (!c || !X_host_in || !X_host_out) return REFINE_E_INVALID;
  if (c->sticky != REFINE_OK) return c->sticky;
  const size_t bytes = (size_t)c->n_loc * c->k * sizeof(double);
  if (!c->dX) RF_CK(c, cudaMalloc(&c->dX, bytes));
  // Dense single rank with the TMA GEMM and >= 1 MiB of X^: upload in chunks on a copy stream while S1
  // runs (its producer warps wait per K step for their chunk; REFINE_H2D_OVERLAP=0 disables); chunks
  // are issued split-interleaved so every split-K CTA's first rows arrive first.
  const bool ov_env = !(getenv("REFINE_H2D_OVERLAP") && getenv("REFINE_H2D_OVERLAP")[0] == '0');
  const bool ov = ov_env && !c->csr && !c->multi && !c->loopback && c->oz_ns == 0 && !c->opts.square &&
                  c->gemm_tma && bytes >= ((size_t)1 << 20) && c->kchunk > 0;
  refine_status st;
  if (ov) {
    constexpr int H2D_MAX_CHUNKS = 64;
    if (!c->h2d) {
      RF_CK(c, cudaStreamCreateWithFlags(&c->h2d, cudaStreamNonBlocking));
      RF_CK(c, cudaEventCreateWithFlags(&c->ev_h2d, cudaEventDisableTiming));
      RF_CK(c, cudaEventCreateWithFlags(&c->ev_pre, cudaEventDisableTiming));
      RF_CK(c, cudaMalloc(&c->h2d_ready, H2D_MAX_CHUNKS * sizeof(unsigned)));
      RF_CK(c, cudaMemsetAsync(c->h2d_ready, 0, H2D_MAX_CHUNKS * sizeof(unsigned), c->stream));
      RF_CK(c, cudaMallocHost(&c->h2d_epoch_host, sizeof(unsigned)));
    }
    // (the previous call ended with a host sync, so its flag copies have read h2d_epoch_host)
    if (++c->h2d_epoch == 0) ++c->h2d_epoch;
    *c->h2d_epoch_host = c->h2d_epoch;
    const int64_t n = c->n_loc, k = c->k;
    const int64_t per_split = std::max<int64_t>(c->kchunk, 16);
    // chunks of `rows` rows aligned globally, `rows` a multiple of 16 (one TMA K step) dividing the split's
    // rows so that no chunk straddles two splits: 4 per split where that divides, else fewer
    int64_t rows = per_split;
    for (int d : {4, 2})
      if (per_split % (16 * d) == 0) { rows = per_split / d; break; }
    if (rows % 16 != 0 || (n + rows - 1) / rows > H2D_MAX_CHUNKS) rows = 0;
    if (rows == 0) {   // (no suitable chunking: plain upload)
      RF_CK(c, cudaMemcpyAsync(c->dX, X_host_in, bytes, cudaMemcpyHostToDevice, c->stream));
      st = launch_sweep(c, c->dX);
      if (st != REFINE_OK) return st;
      RF_CK(c, cudaMemcpyAsync(X_host_out, c->dX, bytes, cudaMemcpyDeviceToHost, c->stream));
      int ds0 = 0;
      if ((st = read_stats(c, stats, &ds0)) != REFINE_OK) return st;
      return map_status(ds0);
    }
    c->h2d_rows = (int)rows;
    RF_CK(c, cudaEventRecord(c->ev_pre, c->stream));   // after earlier work on dX
    RF_CK(c, cudaStreamWaitEvent(c->h2d, c->ev_pre, 0));
    const int64_t cps = (per_split + rows - 1) / rows;   // chunks per split (the last split may have fewer)
    const int64_t nch = (n + rows - 1) / rows;
    for (int64_t p = 0; p < cps; ++p)
      for (int64_t sp = 0; sp * per_split < n; ++sp) {
        const int64_t r0 = sp * per_split + p * rows;
        const int64_t r1 = std::min(std::min(r0 + rows, (sp + 1) * per_split), n);
        if (r0 >= r1) continue;
        const int64_t ch = r0 / rows;   // (rows divides per_split: r0 is chunk-aligned)
        if (ch >= nch) continue;
        RF_CK(c, cudaMemcpyAsync(c->dX + r0 * k, X_host_in + r0 * k, (size_t)(r1 - r0) * k * 8, cudaMemcpyHostToDevice, c->h2d));
        RF_CK(c, cudaMemcpyAsync(c->h2d_ready + ch, c->h2d_epoch_host, sizeof(unsigned), cudaMemcpyHostToDevice, c->h2d));
      }
    RF_CK(c, cudaEventRecord(c->ev_h2d, c->h2d));
    c->h2d_on = true;
    st = enqueue_sweep(c, c->dX);   // (direct launches: the flags' epoch changes per call)
    c->h2d_on = false;
  } else {
    RF_CK(c, cudaMemcpyAsync(c->dX, X_host_in, bytes, cudaMemcpyHostToDevice, c->stream));
    st = launch_sweep(c, c->dX);
  }
  if (st != REFINE_OK) return st;
  RF_CK(c, cudaMemcpyAsync(X_host_out, c->dX, bytes, cudaMemcpyDeviceToHost, c->stream));
  int ds = 0;
  if ((st = read_stats(c, stats, &ds)) != REFINE_OK) return st;
  return map_status(ds);
}

// The sweep loop of refine_run as one CUDA graph with a conditional WHILE node (single rank).  Returns
// false (nothing enqueued, error state cleared) if the graph cannot be built, so the caller falls
// back to enqueuing iters sweeps.
static bool run_as_graph(refine_ctx* c, double* X, int32_t iters, double tol, bool reorth) {
  if (c->multi || c->loopback || getenv("REFINE_RUN_NO_GRAPH")) return false;
  if (!c->cap_stream && cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking) != cudaSuccess) return false;
  cudaGraph_t g = nullptr;
  cudaGraphExec_t ge = nullptr;
  bool ok = false;
  do {
    if (cudaGraphCreate(&g, 0) != cudaSuccess) break;
    cudaGraphConditionalHandle h;
    if (cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault) != cudaSuccess) break;
    cudaGraphNodeParams np = {};
    np.type = cudaGraphNodeTypeConditional;
    np.conditional.handle = h;
    np.conditional.type = cudaGraphCondTypeWhile;
    np.conditional.size = 1;
    cudaGraphNode_t node;
    if (cudaGraphAddNode(&node, g, nullptr, 0, &np) != cudaSuccess) break;
    cudaGraph_t body = np.conditional.phGraph_out[0];
    if (cudaStreamBeginCaptureToGraph(c->cap_stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal) !=
        cudaSuccess)
      break;
    cudaStream_t user = c->stream;
    c->stream = c->cap_stream;
    refine_status st = enqueue_phases(c, X);
    run_cond_kernel<<<1, 1, 0, c->stream>>>(c->ws.status, c->run, c->ws.stats, tol, c->opts.guard_window,
                                            c->opts.guard_factor, c->opts.resid_tol, c->opts.reorth_tol,
                                            reorth ? c->ws.gate : nullptr, iters, h);
    if (st == REFINE_OK && reorth) st = enqueue_rr(c, X, 1, true);
    c->stream = user;
    cudaGraph_t cap = nullptr;
    const cudaError_t e = cudaStreamEndCapture(c->cap_stream, &cap);
    if (st != REFINE_OK || e != cudaSuccess) break;
    if (cudaGraphInstantiate(&ge, g, 0) != cudaSuccess) break;
    ok = cudaGraphLaunch(ge, c->stream) == cudaSuccess;
  } while (0);
  if (ge) cudaGraphExecDestroy(ge);     // (destruction is deferred until the launch completes)
  if (g) cudaGraphDestroy(g);
  if (!ok) {
    cudaGetLastError();                 // clear a non-sticky error from the attempt
    c->sticky = REFINE_OK;
  }
  return ok;
}

extern "C" refine_status refine_run(refine_ctx* c, double* X, int32_t iters, double tol, int32_t* iters_done,
                                    refine_sweep_stats* last) {
  if (!c || !X || iters < 0) return REFINE_E_INVALID;
  if (c->sticky != REFINE_OK) return c->sticky;
  std::vector<refine_ctx*> ranks = c->loopback ? c->kids : std::vector<refine_ctx*>{c};
  for (auto* r : ranks) {
    RF_CK(c, cudaMemsetAsync(r->run, 0, sizeof(RunState), c->stream));
    RF_CK(c, cudaMemsetAsync(r->ws.status, 0, sizeof(int), c->stream));
  }
  // reorthogonalisation policy: single rank -- behind a device gate, no host sync;
  const bool reorth = c->opts.reorth_tol > 0.0 && !c->multi;
  // world > 1: the gated pipeline's collectives cannot be skipped on the device, so the host reads the
  // gate after each sweep (one synchronisation per sweep, only with the policy on) and enqueues the
  // Cholesky-QR step when it is open -- every rank reads the same broadcast statistics: same decision
  const bool reorth_host = c->opts.reorth_tol > 0.0 && c->multi;
  const bool graphed = iters > 0 && run_as_graph(c, X, iters, tol, reorth);
  for (int t = 0; t < iters && !graphed; ++t) {
    refine_status st = enqueue_phases(c, X);
    if (st != REFINE_OK) return st;
    for (auto* r : ranks)      // every rank holds the same stats after the broadcast: same decision
      run_check_kernel<<<1, 1, 0, c->stream>>>(r->ws.status, r->run, r->ws.stats, tol, c->opts.guard_window,
                                               c->opts.guard_factor, c->opts.resid_tol, c->opts.reorth_tol,
                                               (reorth || reorth_host) ? r->ws.gate : nullptr);
    if (reorth && (st = enqueue_rr(c, X, 1, true)) != REFINE_OK) return st;
    if (reorth_host) {
      int h[2] = {0, 0};
      RF_CK(c, cudaMemcpyAsync(&h[0], ctx0(c)->ws.status, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
      RF_CK(c, cudaMemcpyAsync(&h[1], ctx0(c)->ws.gate, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
      RF_CK(c, cudaStreamSynchronize(c->stream));
      if (h[0] != ST_OK) break;
      if (h[1] == ST_OK && (st = enqueue_rr(c, X, 1, false)) != REFINE_OK) return st;
    }
    RF_CK(c, cudaGetLastError());
  }
  RunState rs;
  RF_CK(c, cudaMemcpyAsync(&rs, ctx0(c)->run, sizeof(rs), cudaMemcpyDeviceToHost, c->stream));
  int ds = 0;
  refine_sweep_stats st{};
  refine_status r = read_stats(c, &st, &ds);
  if (r != REFINE_OK) return r;
  int done = rs.done;
  if (ds == ST_DIVERGED && rs.guard && c->opts.rr_fallback) {
    // the correction grew rapidly -- switch to Rayleigh-Ritz preprocessing and
    // continue with its iterations (RR + top-zero sweep) for the remaining budget
    for (; done < iters; ) {
      refine_status q = refine_sweep_rr(c, X, &st, nullptr);
      ++done;
      if (q != REFINE_OK) {
        if (iters_done) *iters_done = done;
        if (last) *last = st;
        return q;
      }
      if (!std::isfinite(st.corr_norm)) { ds = ST_DIVERGED; break; }
      if (st.corr_norm <= tol || (c->opts.resid_tol > 0.0 && st.rel_resid <= c->opts.resid_tol)) {
        ds = ST_HALT_CONVERGED;
        break;
      }
      ds = ST_OK;
    }
  }
  if (iters_done) *iters_done = done;
  if (last) *last = st;
  if (ds == ST_HALT_CONVERGED) return REFINE_OK;
  if (ds == ST_OK) return REFINE_MAXITER;
  return map_status(ds);
}

extern "C" refine_status refine_get_status(refine_ctx* c) {
  if (!c) return REFINE_E_INVALID;
  if (c->sticky != REFINE_OK) return c->sticky;
  int ds = 0;
  RF_CK(c, cudaMemcpyAsync(&ds, ctx0(c)->ws.status, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  RF_CK(c, cudaStreamSynchronize(c->stream));
  return map_status(ds == ST_HALT_CONVERGED ? ST_OK : ds);
}

extern "C" refine_status refine_set_graph(refine_ctx* c, int32_t enable) {
  if (!c) return REFINE_E_INVALID;
  c->use_graph = enable != 0;   // (loopback and NCCL ranks too: the collectives are captured with the kernels)
  if (!c->use_graph && c->gexec) { cudaGraphExecDestroy(c->gexec); c->gexec = nullptr; c->gX = nullptr; }
  return REFINE_OK;
}

extern "C" int32_t refine_kernels_per_sweep(const refine_ctx* c) {
  if (!c) return 0;
  if (c->loopback) {
    int n = 0;
    for (auto* kid : c->kids) n += refine_kernels_per_sweep(kid);
    return n;
  }
  const int per = ((c->csr || c->wfuse) ? 7 : 8) + (c->oz_ns > 0 ? 2 : 0);   // incl. kxk_lu (side stream); emul S1: X slicing; w_finish unless fused
  if (!c->multi) return per;
  return per + 1 - (c->rank == 0 ? 0 : 2);   // + ag_local; kxk_lu / kxk_finish on rank 0 only
}

static const char* kernel_names_dense[] = {"gemm_ax", "w_finish", "kxk_rq", "passB", "passB_reduce",
                                           "kxk_finish", "passC"};
static const char* kernel_names_csr[] = {"spmm_csr", "kxk_rq", "passB", "passB_reduce", "kxk_finish", "passC"};

extern "C" const char* refine_kernel_name(const refine_ctx* c, int32_t i) {
  if (!c || i < 0 || i >= (c->csr ? 6 : 7)) return "";
  return c->csr ? kernel_names_csr[i] : kernel_names_dense[i];
}

extern "C" refine_status refine_profile_begin(refine_ctx* c, int32_t max_sweeps) {
  if (!c || max_sweeps < 1) return REFINE_E_INVALID;
  if (c->loopback) return REFINE_E_UNSUPPORTED;
  if (c->use_graph) return REFINE_E_UNSUPPORTED;      // events are recorded at enqueue time
  if (c->prof_ev) return REFINE_E_INVALID;
  c->prof_per_sweep = (c->csr ? 6 : 7) + 1;   // kernel slots (mark() positions)
  c->prof_cap = c->prof_per_sweep * max_sweeps;
  c->prof_ev = new (std::nothrow) cudaEvent_t[c->prof_cap];
  if (!c->prof_ev) return REFINE_E_NOMEM;
  for (int i = 0; i < c->prof_cap; ++i) RF_CK(c, cudaEventCreate(&c->prof_ev[i]));
  c->prof_used = 0;
  c->prof_max_sweeps = max_sweeps;
  return REFINE_OK;
}

extern "C" refine_status refine_profile_end(refine_ctx* c, double* ms_sum, int32_t* nkernels, int32_t* nsweeps) {
  if (!c || !c->prof_ev) return REFINE_E_INVALID;
  RF_CK(c, cudaStreamSynchronize(c->stream));
  const int per = c->prof_per_sweep, nk = per - 1;
  const int sweeps = c->prof_used / per;
  for (int i = 0; i < nk; ++i) ms_sum[i] = 0.0;
  for (int s = 0; s < sweeps; ++s)
    for (int i = 0; i < nk; ++i) {
      float ms = 0.f;
      RF_CK(c, cudaEventElapsedTime(&ms, c->prof_ev[s * per + i], c->prof_ev[s * per + i + 1]));
      ms_sum[i] += ms;
    }
  for (int i = 0; i < c->prof_cap; ++i) cudaEventDestroy(c->prof_ev[i]);
  delete[] c->prof_ev;
  c->prof_ev = nullptr;
  c->prof_cap = c->prof_used = 0;
  if (nkernels) *nkernels = nk;
  if (nsweeps) *nsweeps = sweeps;
  return REFINE_OK;
}

extern "C" void refine_destroy(refine_ctx* c) {
  if (!c) return;
  if (c->stream) cudaStreamSynchronize(c->stream);
  for (auto* kid : c->kids) refine_destroy(kid);
  c->kids.clear();
  if (c->comm && nccl().ok) nccl().CommDestroy(c->comm);
  if (c->own_xfull && c->Xfull) cudaFree(c->Xfull);
  if (c->Tfull) cudaFree(c->Tfull);
  if (c->ws.halo) cudaFree(c->ws.halo);
  if (c->xoff_buf) cudaFree(c->xoff_buf);
  if (c->st_meta) cudaFree(c->st_meta);
  if (c->gexec) cudaGraphExecDestroy(c->gexec);
  if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
  if (c->side) cudaStreamDestroy(c->side);
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  if (c->pool) cudaFree(c->pool);
  if (c->ws.tlog) cudaFree(c->ws.tlog);
  if (c->dX) cudaFree(c->dX);
  if (c->h2d) cudaStreamDestroy(c->h2d);
  if (c->ev_h2d) cudaEventDestroy(c->ev_h2d);
  if (c->ev_pre) cudaEventDestroy(c->ev_pre);
  if (c->h2d_ready) cudaFree(c->h2d_ready);
  if (c->h2d_epoch_host) cudaFreeHost(c->h2d_epoch_host);
  if (c->oz_e) cudaFree(c->oz_e);
  if (c->oz_diag) cudaFree(c->oz_diag);
  if (c->oz_f) cudaFree(c->oz_f);
  if (c->oz_A) cudaFree(c->oz_A);
  if (c->oz_X) cudaFree(c->oz_X);
  delete c;
}

extern "C" const char* refine_status_string(refine_status s) {
  switch (s) {
    case REFINE_OK: return "REFINE_OK";
    case REFINE_MAXITER: return "REFINE_MAXITER";
    case REFINE_DIVERGED: return "REFINE_DIVERGED";
    case REFINE_E_INVALID: return "REFINE_E_INVALID";
    case REFINE_E_NEAR_ZERO_RQ: return "REFINE_E_NEAR_ZERO_RQ";
    case REFINE_E_ZERO_PIVOT: return "REFINE_E_ZERO_PIVOT";
    case REFINE_E_CUDA: return "REFINE_E_CUDA";
    case REFINE_E_NCCL: return "REFINE_E_NCCL";
    case REFINE_E_NOMEM: return "REFINE_E_NOMEM";
    case REFINE_E_UNSUPPORTED: return "REFINE_E_UNSUPPORTED";
  }
  return "REFINE_UNKNOWN";
}

extern "C" refine_status refine_nccl_id(void* out128) {
  if (!out128) return REFINE_E_INVALID;
  Nccl& N = nccl();
  if (!N.ok) return REFINE_E_NCCL;
  ncclUniqueId id;
  if (N.GetUniqueId(&id) != ncclSuccess) return REFINE_E_NCCL;
  memcpy(out128, &id, sizeof(id));
  return REFINE_OK;
}

extern "C" int32_t refine_halo_plan(int32_t world, int32_t rank, const int64_t* row_begin, const int64_t* row_end,
                                    const int64_t* col_lo, const int64_t* col_hi, int64_t* send, int32_t* nsend,
                                    int64_t* recv, int32_t* nrecv, int64_t* halo_rows, int32_t cap) {
  if (world < 1 || rank < 0 || rank >= world || !row_begin || !row_end || !col_lo || !col_hi) return REFINE_E_INVALID;
  std::vector<refine_ctx::Seg> sv, rv;
  int64_t hr = 0;
  halo_plan(world, rank, row_begin, row_end, col_lo, col_hi, sv, rv, &hr);
  if ((int)sv.size() > cap || (int)rv.size() > cap) return REFINE_E_INVALID;
  for (size_t i = 0; i < sv.size(); ++i) {
    send[4 * i] = sv[i].peer; send[4 * i + 1] = sv[i].row; send[4 * i + 2] = sv[i].cnt; send[4 * i + 3] = sv[i].off;
  }
  for (size_t i = 0; i < rv.size(); ++i) {
    recv[4 * i] = rv[i].peer; recv[4 * i + 1] = rv[i].row; recv[4 * i + 2] = rv[i].cnt; recv[4 * i + 3] = rv[i].off;
  }
  *nsend = (int32_t)sv.size();
  *nrecv = (int32_t)rv.size();
  if (halo_rows) *halo_rows = hr;
  return REFINE_OK;
}

extern "C" refine_status refine_debug_get(refine_ctx* c, int32_t what, double* dst) {
  if (!c || !dst) return REFINE_E_INVALID;
  if (c->sticky != REFINE_OK) return c->sticky;
  if (c->loopback) return refine_debug_get(c->kids[0], what, dst);   // rank 0 holds the k x k state
  const int k = c->k;
  const size_t kk = (size_t)k * k, nk = (size_t)c->n_loc * k;
  const Ws& ws = c->ws;
  const double* src = nullptr;
  size_t cnt = 0;
  switch (what) {
    case 0: src = ws.W; cnt = nk; break;
    case 1: src = ws.sigma; cnt = k; break;
    case 2: src = ws.U; cnt = kk; break;
    case 3: src = ws.L; cnt = kk; break;
    case 4: src = ws.T; cnt = kk; break;
    case 5: src = ws.d; cnt = k; break;
    case 6: src = ws.alpha; cnt = k; break;
    case 7: src = ws.E11; cnt = kk; break;
    case 8:
      trsm_y_kernel<<<c->sms * 4, 128, 0, c->stream>>>(c->ws, dst);
      RF_CK(c, cudaGetLastError());
      RF_CK(c, cudaStreamSynchronize(c->stream));
      return REFINE_OK;
    case 9: src = ws.stats; cnt = 8; break;
    case 11: {  // S1 kernel geometry: [stencil on, R, L, nq, grid, nx, ny, nz, gather R]
      const StencilGeo& g = c->st_geo;
      const double h[9] = {c->st_on ? 1.0 : 0.0, (double)g.R, (double)g.L, (double)g.nq, (double)c->st_grid,
                           (double)g.nx, (double)g.ny, (double)g.nz, (double)c->gather_R};
      RF_CK(c, cudaMemcpyAsync(dst, h, sizeof(h), cudaMemcpyHostToDevice, c->stream));
      RF_CK(c, cudaStreamSynchronize(c->stream));
      return REFINE_OK;
    }
    case 10:   // clock64 phase log (REFINE_KXK_TIMING=1), raw int64 bits
      if (!ws.tlog) return REFINE_E_UNSUPPORTED;
      src = reinterpret_cast<const double*>(ws.tlog); cnt = 64; break;
    default: return REFINE_E_INVALID;
  }
  RF_CK(c, cudaMemcpyAsync(dst, src, cnt * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  RF_CK(c, cudaStreamSynchronize(c->stream));
  return REFINE_OK;
}
