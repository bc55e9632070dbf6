// refine.cu -- host runtime and C ABI (include/refine.h) of the B200-native refinement sweep.
//
// One sweep = the launch sequence below on the caller's stream:
//   dense: gemm_ax (DMMA, split-K) -> w_finish            | CSR: spmm_csr (fma chain, fused)
//   kxk_prep -> passB -> passB_reduce -> kxk_finish -> passC -> norm_reduce -> normalize
// Device-side conditions are carried by a status word every kernel checks first, so a
// failed or halted sweep leaves X untouched and refine_run needs no per-sweep host sync.
#include <cuda_runtime.h>

#include <algorithm>
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

using namespace rf;

namespace {

constexpr int ST_HALT_CONVERGED = 100;   // refine_run: device-side stop (converged)

struct RunState {   // device-resident refine_run bookkeeping
  int32_t done;     // sweeps completed
  int32_t pad;
  double hist[4];   // last corr norms (ring) for the divergence guard
};

__global__ void run_check_kernel(int* status, RunState* rs, const double* stats, double tol, int window,
                                 double factor) {
  if (*status != ST_OK) return;
  const double c = stats[1];
  const int t = rs->done;
  rs->done = t + 1;
  if (!isfinite(c)) { *status = ST_DIVERGED; return; }
  if (c <= tol) { *status = ST_HALT_CONVERGED; return; }
  if (window > 0 && window <= 4 && t >= window && c >= factor * rs->hist[(t - window) & 3]) {
    *status = ST_DIVERGED;
    return;
  }
  rs->hist[t & 3] = c;
}

__global__ void absrow_max_dense_kernel(const double* A, int64_t lda, int64_t n_loc, int64_t n, int64_t row0,
                                        double shift, double* out_rows) {
  const int lane = threadIdx.x & 31;
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = w; i < n_loc; i += nw) {
    double s = 0.0;
    for (int64_t l = lane; l < n; l += 32) {
      double a = A[i * lda + l];
      if (l == row0 + i) a -= shift;
      s += fabs(a);
    }
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) out_rows[i] = s;
  }
}
__global__ void absrow_max_csr_kernel(const int32_t* rp, const int32_t* ci, const double* v, int64_t n_loc,
                                      int64_t row0, double shift, double* out_rows) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_loc; i += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    bool diag = false;
    for (int32_t p = rp[i] - rp[0]; p < rp[i + 1] - rp[0]; ++p) {
      double a = v[p];
      if (ci[p] == row0 + i) { a -= shift; diag = true; }
      s += fabs(a);
    }
    if (!diag) s += fabs(shift);
    out_rows[i] = s;
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
  double shift = 0.0;
  refine_opts opts{};
  int rank = 0, world = 1;
  Ws ws{};
  void* pool = nullptr;
  size_t pool_bytes = 0;
  // dense GEMM launch
  int gemm_bm = 0, nsplit = 1;
  int64_t kchunk = 0;
  int gemm_gx = 0;
  int n_ag = 0, w_fin_grid = 0, spmm_grid = 0;
  int passb_grid_y = 0, passc_grid = 0;
  RunState* run = nullptr;
  refine_status sticky = REFINE_OK;
  // graph
  bool use_graph = false;
  cudaGraphExec_t gexec = nullptr;
  double* gX = nullptr;
  cudaStream_t cap_stream = nullptr;   // graphs are captured on a private stream (the caller's may be legacy)
  // host-buffer entry point
  double* dX = nullptr;
  int launches = 0;
  // live per-kernel timing (refine_profile_begin/end): events at every kernel boundary
  cudaEvent_t* prof_ev = nullptr;
  int prof_cap = 0, prof_used = 0, prof_per_sweep = 0, prof_sweeps = 0, prof_max_sweeps = 0;
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

// ---------------------------------------------------------------- per-KP kernel tables
template <int KP> struct Tiles;
//                 GEMM: BM  WM  WN  BK  ST | passB: TA  TB  WA WB  BR | passC: NC BM WM WN
template <> struct Tiles<8>   { static constexpr int G[5] = {64, 16, 8, 32, 4};   static constexpr int B[5] = {8, 16, 1, 2, 32};   static constexpr int C[4] = {8, 64, 8, 1}; };
template <> struct Tiles<16>  { static constexpr int G[5] = {64, 16, 16, 32, 4};  static constexpr int B[5] = {16, 32, 2, 4, 32};  static constexpr int C[4] = {16, 64, 8, 1}; };
template <> struct Tiles<32>  { static constexpr int G[5] = {128, 32, 16, 32, 2}; static constexpr int B[5] = {32, 64, 2, 4, 32};  static constexpr int C[4] = {32, 64, 4, 2}; };
template <> struct Tiles<64>  { static constexpr int G[5] = {128, 64, 16, 32, 2}; static constexpr int B[5] = {64, 128, 2, 4, 16}; static constexpr int C[4] = {64, 64, 2, 4}; };
template <> struct Tiles<128> { static constexpr int G[5] = {64, 32, 32, 32, 2};  static constexpr int B[5] = {64, 64, 2, 4, 16};  static constexpr int C[4] = {64, 16, 1, 8}; };

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
  static constexpr auto passB = passB_kernel<KP, BTA, BTB, BWA, BWB, BBR>;
  static constexpr auto passBred = passB_reduce_kernel<KP, BTA, BTB, BWA, BWB, BBR>;
  static constexpr auto passC = passC_kernel<KP, CNC, CBM, CWM, CWN>;

  static cudaError_t setup(refine_ctx* c) {
    cudaError_t e;
    if ((e = cudaFuncSetAttribute(gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, GC::SMEM))) return e;
    if ((e = cudaFuncSetAttribute(passB, cudaFuncAttributeMaxDynamicSharedMemorySize, BC::SMEM))) return e;
    if ((e = cudaFuncSetAttribute(passC, cudaFuncAttributeMaxDynamicSharedMemorySize, CC::SMEM))) return e;
    int occ = 1;
    // dense GEMM: split-K so the grid fills whole waves of resident CTAs
    if (!c->csr) {
      if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, gemm, GC::THREADS, GC::SMEM))) return e;
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
      c->nsplit = best;
      const int64_t kit = (kiters + best - 1) / best;
      c->kchunk = kit * GBK;
      c->nsplit = (int)((c->n + c->kchunk - 1) / c->kchunk);
    }
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, passB, BC::THREADS, BC::SMEM))) return e;
    occ = std::max(occ, 1);
    const int64_t rows = std::max<int64_t>(c->n_loc - c->ws.top, 1);
    const int64_t max_chunks = std::max<int64_t>((rows + 255) / 256, 1);   // >= 256 rows per chunk
    c->passb_grid_y = (int)std::min<int64_t>(std::max(c->sms * occ / BC::NTILES, 1), max_chunks);
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, passC, CC::THREADS, CC::SMEM))) return e;
    occ = std::max(occ, 1);
    const int64_t ctiles = std::max<int64_t>((rows + CBM - 1) / CBM, 1);
    c->passc_grid = (int)std::min<int64_t>(std::max(c->sms * occ / (KP / CNC), 1), ctiles);
    return cudaSuccess;
  }

  static void sizes(refine_ctx* c, size_t& bpart, size_t& brr, size_t& nslot) {
    bpart = (size_t)c->passb_grid_y * BC::NTILES * BTA * BTB;
    brr = (size_t)c->passb_grid_y * KP;
    nslot = (size_t)c->passc_grid * KP;
  }

  static int enqueue(refine_ctx* c, double* X) {
    Ws& ws = c->ws;
    cudaStream_t s = c->stream;
    int n = 0;
    const bool xv16 = (c->k % 2 == 0) && ((uintptr_t)X % 16 == 0);
    if (!c->csr) {
      const bool av16 = (c->n % 2 == 0) && (c->lda % 2 == 0) && ((uintptr_t)c->A % 16 == 0) && (c->kchunk % 2 == 0);
      double* out = (c->nsplit == 1) ? ws.W : ws.Wpart;
      c->mark();
      gemm<<<dim3(c->gemm_gx, c->nsplit), GC::THREADS, GC::SMEM, s>>>(
          c->A, c->lda, X, c->k, c->n_loc, c->n, c->kchunk, out, c->n_loc * c->k, av16, xv16, ws.status);
      c->mark();
      w_finish_kernel<<<c->w_fin_grid, 256, 0, s>>>(ws, X, c->nsplit, c->n_loc * c->k);
      n += 2;
    } else {
      c->mark();
      const bool vec = xv16 && (c->k & (c->k - 1)) == 0 && c->k >= 2;
      auto* Xg = X;
      if (vec) {
        switch (c->k) {
          case 2: spmm_csr_vec_kernel<1, 1><<<c->spmm_grid, 256, 0, s>>>(ws, c->rp, c->ci, c->val, Xg, X); break;
          case 4: spmm_csr_vec_kernel<1, 2><<<c->spmm_grid, 256, 0, s>>>(ws, c->rp, c->ci, c->val, Xg, X); break;
          case 8: spmm_csr_vec_kernel<1, 4><<<c->spmm_grid, 256, 0, s>>>(ws, c->rp, c->ci, c->val, Xg, X); break;
          case 16: spmm_csr_vec_kernel<1, 8><<<c->spmm_grid, 256, 0, s>>>(ws, c->rp, c->ci, c->val, Xg, X); break;
          case 32: spmm_csr_vec_kernel<1, 16><<<c->spmm_grid, 256, 0, s>>>(ws, c->rp, c->ci, c->val, Xg, X); break;
          case 64: spmm_csr_vec_kernel<1, 32><<<c->spmm_grid, 256, 0, s>>>(ws, c->rp, c->ci, c->val, Xg, X); break;
          default: spmm_csr_vec_kernel<2, 32><<<c->spmm_grid, 256, 0, s>>>(ws, c->rp, c->ci, c->val, Xg, X); break;
        }
      } else {
        switch ((c->k + 31) / 32) {
          case 1: spmm_csr_kernel<1><<<c->spmm_grid, 256, 0, s>>>(ws, c->rp, c->ci, c->val, Xg, X); break;
          case 2: spmm_csr_kernel<2><<<c->spmm_grid, 256, 0, s>>>(ws, c->rp, c->ci, c->val, Xg, X); break;
          case 3: spmm_csr_kernel<3><<<c->spmm_grid, 256, 0, s>>>(ws, c->rp, c->ci, c->val, Xg, X); break;
          default: spmm_csr_kernel<4><<<c->spmm_grid, 256, 0, s>>>(ws, c->rp, c->ci, c->val, Xg, X); break;
        }
      }
      n += 1;
    }
    c->mark();
    kxk_prep_kernel<<<1, KXK_THREADS, std::max(c->k <= 64 ? 4 * c->k * c->k : c->k * c->k, PANEL_SMEM) * 8, s>>>(ws, X);
    c->mark();
    passB<<<dim3(BC::NTILES, c->passb_grid_y), BC::THREADS, BC::SMEM, s>>>(ws, X, xv16);
    c->mark();
    passBred<<<(2 * c->k * c->k + c->k + 31) / 32, 256, 0, s>>>(ws, c->passb_grid_y);
    c->mark();
    kxk_finish_kernel<<<1, KXK_THREADS, PANEL_SMEM * 8, s>>>(ws, X, ws.W);
    c->mark();
    passC<<<dim3(c->passc_grid, KP / CNC), CC::THREADS, CC::SMEM, s>>>(ws, X, xv16);
    c->mark();
    norm_reduce_kernel<<<1, 128, 0, s>>>(ws);
    if (c->opts.normalize) {
      c->mark();
      normalize_kernel<<<c->sms * 8, 256, 0, s>>>(ws, X);
      ++n;
    }
    c->mark();
    return n + 6;
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
static refine_status init_common(refine_ctx* c, int64_t n, int32_t k, int64_t row_begin, int64_t row_end,
                                 double shift, const refine_comm* comm, const refine_opts* opts, void* stream) {
  if (k < 1 || (int64_t)k >= n || row_begin < 0 || row_end > n || row_end <= row_begin) return REFINE_E_INVALID;
  if (k > KMAX) return REFINE_E_UNSUPPORTED;
  c->rank = comm ? comm->rank : 0;
  c->world = comm ? comm->world : 1;
  if (c->world != 1) return REFINE_E_UNSUPPORTED;      // multi-GPU row partition: see DESIGN.md
  if (c->rank == 0 && (row_begin != 0 || row_end - row_begin < k)) return REFINE_E_INVALID;
  c->n = n; c->k = k; c->kp = pad_kp(k);
  c->row_begin = row_begin; c->row_end = row_end; c->n_loc = row_end - row_begin;
  c->shift = shift;
  c->opts = refine_opts{10.0, 0, 1, 3, 10.0};
  if (opts) c->opts = *opts;
  c->stream = (cudaStream_t)stream;
  RF_CK(c, cudaGetDevice(&c->device));
  RF_CK(c, cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, c->device));
  Ws& ws = c->ws;
  ws.n_loc = c->n_loc; ws.k = k; ws.kp = c->kp;
  ws.top = (c->rank == 0) ? k : 0;
  ws.shift = shift;
  ws.beta_zero = c->opts.beta_zero;
  refine_status st = REFINE_OK;
  RF_CK(c, (cudaError_t)dispatch(c->kp, [&](auto K) { return decltype(K)::setup(c); }));
  RF_CK(c, cudaFuncSetAttribute(kxk_prep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, std::max(KMAX * KMAX, std::max(PANEL_SMEM, 4 * 64 * 64)) * 8));
  RF_CK(c, cudaFuncSetAttribute(kxk_finish_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, PANEL_SMEM * 8));
  // workspace sizes (doubles)
  size_t bpart = 0, brr = 0, nslot = 0;
  dispatch(c->kp, [&](auto K) { decltype(K)::sizes(c, bpart, brr, nslot); return 0; });
  c->w_fin_grid = (int)std::max<int64_t>(1, std::min<int64_t>(c->sms * 4, c->n_loc / 2));
  c->spmm_grid = (int)std::max<int64_t>(1, std::min<int64_t>(c->sms * 8, (c->n_loc + 7) / 8));
  c->n_ag = c->csr ? c->spmm_grid : c->w_fin_grid;
  const size_t nk = (size_t)c->n_loc * k, kk = (size_t)k * k;
  const size_t wpart = (!c->csr && c->nsplit > 1) ? (size_t)c->nsplit * nk : 0;
  size_t off = 0;
  auto take = [&](size_t cnt) { size_t o = off; off += (cnt + 31) & ~size_t(31); return o; };
  const size_t oW = take(nk), oWp = take(wpart), oAg = take((size_t)c->n_ag * k * 4), oBp = take(bpart),
               oBrr = take(brr), oM2 = take(kk), oG2 = take(kk), oRr = take(k), oNs = take(nslot),
               oAl = take(k), oD = take(k), oRd = take(k), oSg = take(k), oU = take(kk), oL = take(kk),
               oT = take(kk), oUi = take(kk), oE = take(kk), oCs = take(kk), oSc = take(k), oNt = take(k), oIn = take(k),
               oSt = take(8), oScr = take(16 * kk), oRows = take((size_t)c->n_loc), oRun = take(8);
  const size_t bytes = off * 8 + 64;
  RF_CK(c, cudaMalloc(&c->pool, bytes));
  c->pool_bytes = bytes;
  RF_CK(c, cudaMemsetAsync(c->pool, 0, bytes, c->stream));
  double* b = (double*)c->pool;
  ws.W = b + oW; ws.Wpart = wpart ? b + oWp : nullptr; ws.ag = b + oAg; ws.n_ag = c->n_ag;
  ws.bpart = b + oBp; ws.brr = b + oBrr; ws.n_chunk = c->passb_grid_y;
  ws.M2 = b + oM2; ws.G2 = b + oG2; ws.rr2 = b + oRr; ws.nslot = b + oNs; ws.n_nslot = c->passc_grid;
  ws.alpha = b + oAl; ws.d = b + oD; ws.rd = b + oRd; ws.sigma = b + oSg; ws.U = b + oU; ws.L = b + oL;
  ws.T = b + oT; ws.Uinv = b + oUi; ws.E11 = b + oE; ws.Csig = b + oCs; ws.scal = b + oSc; ws.ntop = b + oNt; ws.invn = b + oIn;
  ws.stats = b + oSt; ws.scratch = b + oScr;
  c->run = reinterpret_cast<RunState*>(b + oRun);
  ws.status = reinterpret_cast<int*>(b + off);     // after all arrays (64 spare bytes)
  ws.tlog = nullptr;
  if (getenv("REFINE_KXK_TIMING")) RF_CK(c, cudaMalloc(&ws.tlog, 64 * sizeof(long long)));
  // ||A - shift I||_inf (one pass over A) -> delta = c ||A|| u
  double* rows = b + oRows;
  if (!c->csr)
    absrow_max_dense_kernel<<<c->sms * 8, 256, 0, c->stream>>>(c->A, c->lda, c->n_loc, c->n, c->row_begin, shift, rows);
  else
    absrow_max_csr_kernel<<<c->sms * 8, 256, 0, c->stream>>>(c->rp, c->ci, c->val, c->n_loc, c->row_begin, shift, rows);
  max_kernel<<<1, 1024, 0, c->stream>>>(rows, c->n_loc, ws.stats + 7);
  RF_CK(c, cudaGetLastError());
  double normA = 0.0;
  RF_CK(c, cudaMemcpyAsync(&normA, ws.stats + 7, 8, cudaMemcpyDeviceToHost, c->stream));
  RF_CK(c, cudaStreamSynchronize(c->stream));
  ws.normA = normA;
  ws.delta = c->opts.delta_c * normA * std::ldexp(1.0, -53);
  return st;
}

extern "C" refine_status refine_init_dense(refine_ctx** out, int64_t n, int32_t k, const double* A_rows, int64_t lda,
                                           int64_t row_begin, int64_t row_end, double shift,
                                           const refine_comm* comm, const refine_opts* opts, void* stream) {
  if (!out) return REFINE_E_INVALID;
  *out = nullptr;
  if (!A_rows || lda < n) return REFINE_E_INVALID;
  refine_ctx* c = new (std::nothrow) refine_ctx();
  if (!c) return REFINE_E_NOMEM;
  c->csr = false; c->A = A_rows; c->lda = lda;
  refine_status st = init_common(c, n, k, row_begin, row_end, shift, comm, opts, stream);
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
  c->csr = true; c->rp = row_ptr; c->ci = col_idx; c->val = val;
  refine_status st = init_common(c, n, k, row_begin, row_end, shift, comm, opts, stream);
  if (st != REFINE_OK) { refine_destroy(c); return st; }
  *out = c;
  return REFINE_OK;
}

// ---------------------------------------------------------------- sweeps
static refine_status enqueue_sweep(refine_ctx* c, double* X) {
  RF_CK(c, cudaMemsetAsync(c->ws.status, 0, sizeof(int), c->stream));
  c->launches = dispatch(c->kp, [&](auto K) { return decltype(K)::enqueue(c, X); });
  RF_CK(c, cudaGetLastError());
  return REFINE_OK;
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
    refine_status st = enqueue_sweep(c, X);
    c->stream = user;
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
  RF_CK(c, cudaMemcpyAsync(h, c->ws.stats, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
  RF_CK(c, cudaMemcpyAsync(&st, c->ws.status, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  RF_CK(c, cudaStreamSynchronize(c->stream));
  if (stats) {
    stats->rel_resid = h[0]; stats->corr_norm = h[1]; stats->min_gap = h[2];
    stats->delta_hits = (int32_t)h[3]; stats->flipped = (int32_t)h[4];
  }
  *dev_status = st;
  return REFINE_OK;
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
  RF_CK(c, cudaMemcpyAsync(c->dX, X_host_in, bytes, cudaMemcpyHostToDevice, c->stream));
  refine_status st = launch_sweep(c, c->dX);
  if (st != REFINE_OK) return st;
  RF_CK(c, cudaMemcpyAsync(X_host_out, c->dX, bytes, cudaMemcpyDeviceToHost, c->stream));
  int ds = 0;
  if ((st = read_stats(c, stats, &ds)) != REFINE_OK) return st;
  return map_status(ds);
}

extern "C" refine_status refine_run(refine_ctx* c, double* X, int32_t iters, double tol, int32_t* iters_done,
                                    refine_sweep_stats* last) {
  if (!c || !X || iters < 0) return REFINE_E_INVALID;
  if (c->sticky != REFINE_OK) return c->sticky;
  RF_CK(c, cudaMemsetAsync(c->run, 0, sizeof(RunState), c->stream));
  RF_CK(c, cudaMemsetAsync(c->ws.status, 0, sizeof(int), c->stream));
  for (int t = 0; t < iters; ++t) {
    c->launches = dispatch(c->kp, [&](auto K) { return decltype(K)::enqueue(c, X); });
    run_check_kernel<<<1, 1, 0, c->stream>>>(c->ws.status, c->run, c->ws.stats, tol, c->opts.guard_window,
                                             c->opts.guard_factor);
    RF_CK(c, cudaGetLastError());
  }
  RunState rs;
  RF_CK(c, cudaMemcpyAsync(&rs, c->run, sizeof(rs), cudaMemcpyDeviceToHost, c->stream));
  int ds = 0;
  refine_sweep_stats st{};
  refine_status r = read_stats(c, &st, &ds);
  if (r != REFINE_OK) return r;
  if (iters_done) *iters_done = rs.done;
  if (last) *last = st;
  if (ds == ST_HALT_CONVERGED) return REFINE_OK;
  if (ds == ST_OK) return REFINE_MAXITER;
  return map_status(ds);
}

extern "C" refine_status refine_get_status(refine_ctx* c) {
  if (!c) return REFINE_E_INVALID;
  if (c->sticky != REFINE_OK) return c->sticky;
  int ds = 0;
  RF_CK(c, cudaMemcpyAsync(&ds, c->ws.status, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  RF_CK(c, cudaStreamSynchronize(c->stream));
  return map_status(ds == ST_HALT_CONVERGED ? ST_OK : ds);
}

extern "C" refine_status refine_set_graph(refine_ctx* c, int32_t enable) {
  if (!c) return REFINE_E_INVALID;
  c->use_graph = enable != 0;
  if (!c->use_graph && c->gexec) { cudaGraphExecDestroy(c->gexec); c->gexec = nullptr; c->gX = nullptr; }
  return REFINE_OK;
}

extern "C" int32_t refine_kernels_per_sweep(const refine_ctx* c) {
  if (!c) return 0;
  return (c->csr ? 7 : 8) + (c->opts.normalize ? 1 : 0);
}

static const char* kernel_names_dense[] = {"gemm_ax", "w_finish", "kxk_prep", "passB", "passB_reduce",
                                           "kxk_finish", "passC", "norm_reduce", "normalize"};
static const char* kernel_names_csr[] = {"spmm_csr", "kxk_prep", "passB", "passB_reduce",
                                         "kxk_finish", "passC", "norm_reduce", "normalize"};

extern "C" const char* refine_kernel_name(const refine_ctx* c, int32_t i) {
  if (!c || i < 0 || i >= refine_kernels_per_sweep(c)) return "";
  return c->csr ? kernel_names_csr[i] : kernel_names_dense[i];
}

extern "C" refine_status refine_profile_begin(refine_ctx* c, int32_t max_sweeps) {
  if (!c || max_sweeps < 1) return REFINE_E_INVALID;
  if (c->use_graph) return REFINE_E_UNSUPPORTED;      // events are recorded at enqueue time
  if (c->prof_ev) return REFINE_E_INVALID;
  c->prof_per_sweep = refine_kernels_per_sweep(c) + 1;
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
  if (c->gexec) cudaGraphExecDestroy(c->gexec);
  if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
  if (c->pool) cudaFree(c->pool);
  if (c->ws.tlog) cudaFree(c->ws.tlog);
  if (c->dX) cudaFree(c->dX);
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
  return REFINE_E_UNSUPPORTED;   // multi-GPU path not in this build
}

extern "C" refine_status refine_debug_get(refine_ctx* c, int32_t what, double* dst) {
  if (!c || !dst) return REFINE_E_INVALID;
  if (c->sticky != REFINE_OK) return c->sticky;
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
    case 10:   // clock64 phase log (REFINE_KXK_TIMING=1), raw int64 bits
      if (!ws.tlog) return REFINE_E_UNSUPPORTED;
      src = reinterpret_cast<const double*>(ws.tlog); cnt = 64; break;
    default: return REFINE_E_INVALID;
  }
  RF_CK(c, cudaMemcpyAsync(dst, src, cnt * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  RF_CK(c, cudaStreamSynchronize(c->stream));
  return REFINE_OK;
}
