// common.cuh -- device helpers shared by the sweep kernels (sm_100a, FP64).
//
//  * DMMA: the FP64 tensor-core instruction.  sm_100a has no tcgen05 FP64 kind;
//    every f64 mma.sync shape lowers to SASS DMMA.8x8x4 (checked with cuobjdump),
//    so m8n8k4 is used directly.  Measured on the B200 box: 37.1 TFLOP/s chip
//    peak (tools/fp64_peak.cu, profiles/r01_fp64_peaks.json) vs 34.2 for DFMA.
//  * double-double accumulation (error-free TwoSum / TwoProd) for the length-n
//    reductions whose rounding is amplified by 1/gap in eq. (Eoffdiag)
//    (alpha_j and x_j^T w_j).
//  * cp.async (LDGSTS) staging.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#define RF_DEV __device__ __forceinline__

namespace rf {

constexpr int KMAX = 128;       // largest k compiled (BASELINE configs use 4..128)

// ---------------------------------------------------------------- DMMA m8n8k4
// A (8x4, row): thread t holds A[t>>2][t&3];  B (4x8, col): thread t holds B[t&3][t>>2];
// C (8x8): thread t holds C[t>>2][2*(t&3)], C[t>>2][2*(t&3)+1].
RF_DEV void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

// ---------------------------------------------------------------- cp.async
RF_DEV uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
// 1024-byte-aligned start inside a dynamic shared-memory array, derived by integer offset from the
// __shared__ array itself: the compiler then keeps the shared window (LDS / STS) for everything
// addressed through it -- a round trip through uintptr_t makes every access a generic LD / ST
RF_DEV unsigned char* smem_align1024(unsigned char* p) { return p + ((1024u - (smem_u32(p) & 1023u)) & 1023u); }
RF_DEV void cp_async16(void* smem, const void* gmem, bool pred) {
  // src-size 0 zero-fills the 16 bytes
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(smem)), "l"(gmem),
               "r"(pred ? 16 : 0));
}
RF_DEV void cp_async8(void* smem, const void* gmem, bool pred) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(smem)), "l"(gmem),
               "r"(pred ? 8 : 0));
}
RF_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
RF_DEV void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// ---------------------------------------------------------------- programmatic dependent launch
// The sweep's kernels are launched with cudaLaunchAttributeProgrammaticStreamSerialization (refine.cu
// launch_k), so a kernel's CTAs may be scheduled while its predecessor drains; every such kernel
// waits here before touching memory the predecessor writes (a no-op for an ordinary launch).
RF_DEV void griddep_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }

// ---------------------------------------------------------------- mbarrier + bulk / tensor copies
RF_DEV void mbar_init(uint64_t* mbar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(mbar)), "r"(count));
}
RF_DEV void mbar_wait(uint64_t* mbar, uint32_t parity) {
  uint32_t done = 0;
  while (!done)
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(done)
        : "r"(smem_u32(mbar)), "r"(parity)
        : "memory");
}
RF_DEV void mbar_expect_tx(uint64_t* mbar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(mbar)), "r"(bytes) : "memory");
}
RF_DEV void mbar_arrive(uint64_t* mbar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(mbar)) : "memory");
}
// Order this thread's view of prior generic-proxy shared-memory accesses (other threads' reads,
// acquired through an mbarrier wait) before its subsequent async-proxy operations on them (TMA /
// bulk-copy refills of a ring slot, tcgen05 reads of operands stored with st.shared).
RF_DEV void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
// Stage-release counter of the barrier-free rings (stencil SpMM, ping-pong passes B / C): lane 0 of
// a warp whose reads of a stage are done (after __syncwarp) counts itself in with a release atomic;
// returns true for the last of `nw` warps of this use of the stage, which then acquires (so every
// warp's generic reads happen before) and proxy-fences before refilling the stage by TMA.  The
// release / acquire pair compiles to MEMBAR.ALL.CTA (a __threadfence_block is fence.sc, MEMBAR.SC).
RF_DEV bool stage_release_last(int* ctr, int nw) {
  int old;
  asm volatile("atom.release.cta.shared::cta.add.u32 %0, [%1], 1;\n" : "=r"(old) : "r"(smem_u32(ctr)) : "memory");
  if (old % nw != nw - 1) return false;
  asm volatile("fence.acq_rel.cta;\n" ::: "memory");
  fence_async_smem();
  return true;
}
// 1-D bulk copy global -> shared (16-byte aligned, size a multiple of 16), completing on mbar
RF_DEV void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* mbar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(mbar))
               : "memory");
}
// 2-D TMA tile load (box at signed coordinates (c0 = inner, c1)), as tma_load_4d
RF_DEV void tma_load_2d(void* dst, const void* tmap, int c0, int c1, uint64_t* mbar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          smem_u32(dst)),
      "l"(tmap), "r"(c0), "r"(c1), "r"(smem_u32(mbar))
      : "memory");
}
// 4-D TMA tile load (cp.async.bulk.tensor; SASS UTMALDG) of the box at signed coordinates
// (c0..c3) of the tensor map (a __grid_constant__ kernel parameter); elements outside the tensor
// are zero-filled and still counted in the transaction bytes.
RF_DEV void tma_load_4d(void* dst, const void* tmap, int c0, int c1, int c2, int c3, uint64_t* mbar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
      "[%6];\n" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(mbar))
      : "memory");
}
// L2 prefetches (no shared memory, no completion): the box tma_load_4d / tma_load_2d would load, and
// a 1-D range (16-byte aligned, size a multiple of 16).  They put DRAM requests in flight ahead of
// the shared-memory ring, whose depth alone (one or two loads per SM) is too small for HBM latency.
RF_DEV void tma_prefetch_4d(const void* tmap, int c0, int c1, int c2, int c3) {
  asm volatile("cp.async.bulk.prefetch.tensor.4d.L2.global.tile [%0, {%1, %2, %3, %4}];\n" ::"l"(tmap), "r"(c0), "r"(c1),
               "r"(c2), "r"(c3)
               : "memory");
}
RF_DEV void tma_prefetch_2d(const void* tmap, int c0, int c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];\n" ::"l"(tmap), "r"(c0), "r"(c1) : "memory");
}
RF_DEV void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(src), "r"(bytes) : "memory");
}

// ---------------------------------------------------------------- double-double
// Error-free transforms with explicit round-to-nearest intrinsics so that nvcc's
// default fma contraction can never merge the products and sums below.
struct dd { double hi, lo; };
RF_DEV dd two_sum(double a, double b) {
  double s = __dadd_rn(a, b);
  double bb = __dadd_rn(s, -a);
  double e = __dadd_rn(__dadd_rn(a, -__dadd_rn(s, -bb)), __dadd_rn(b, -bb));
  return {s, e};
}
RF_DEV dd quick_two_sum(double a, double b) {
  double s = __dadd_rn(a, b);
  return {s, __dadd_rn(b, -__dadd_rn(s, -a))};
}
// acc += a*b exactly-rounded-to-dd
RF_DEV void dd_add_prod(dd& acc, double a, double b) {
  double p = __dmul_rn(a, b);
  double pe = __fma_rn(a, b, -p);
  dd s = two_sum(acc.hi, p);
  double e = __dadd_rn(s.lo, __dadd_rn(acc.lo, pe));
  acc = quick_two_sum(s.hi, e);
}
RF_DEV void dd_add(dd& acc, dd x) {
  dd s = two_sum(acc.hi, x.hi);
  double e = __dadd_rn(s.lo, __dadd_rn(acc.lo, x.lo));
  acc = quick_two_sum(s.hi, e);
}
RF_DEV double dd_val(dd a) { return __dadd_rn(a.hi, a.lo); }
// acc += x (x a plain double)
RF_DEV void dd_add1(dd& acc, double x) {
  dd s = two_sum(acc.hi, x);
  acc = quick_two_sum(s.hi, __dadd_rn(s.lo, acc.lo));
}

// device status codes (same values as refine_status)
enum : int { ST_OK = 0, ST_DIVERGED = 2, ST_E_INVALID = -1, ST_E_NEAR_ZERO_RQ = -2, ST_E_ZERO_PIVOT = -3 };

// Everything the sweep keeps on the device; passed to kernels by value.
struct Ws {
  int64_t n_loc;     // local rows
  int32_t k, kp;     // k and its padded power-of-two tile width (>= 8)
  int32_t top;       // local rows [0, top) are the top k x k block (k on rank 0, else 0)
  double shift, delta, normA;
  int32_t beta_zero;
  double* W;         // n_loc x k
  double* Xt;        // n_loc x k: X~ (written by kxk_finish / passC, read by normalize)
  double* Wpart;     // split-K partials (dense), S x n_loc x k
  double* ag;        // alpha/g double-double slots: n_ag x k x 4 {a_hi, a_lo, g_hi, g_lo}
  int32_t n_ag;
  double* bpart;     // pass-B partials: n_chunk x tiles x (TA x TB), plus rr: n_chunk x kp
  double* brr;
  int32_t n_chunk;
  double* M2;        // kp x kp  (X_2^T R_2, un-flipped)
  double* G2;        // kp x kp  (X_2^T X_2)
  double* rr2;       // kp       (sum_i r_ij^2 over rows >= top)
  double* nslot;     // norm partial slots: n_nslot x kp
  int32_t n_nslot;
  // k x k state (row-major, ld = k)
  double *alpha, *d, *rd, *sigma, *U, *L, *Uinv, *T, *E11, *Csig, *scal, *ntop, *invn, *stats;
  double* scratch;   // 16 k x k scratch matrices for the k x k algebra
  int* status;
  // row partition (world > 1; world == 1: row0 = 0, row1 = n_loc, halo = nullptr)
  int32_t world, rank;
  int32_t multi;          // 1: the multi-rank code path (gathered partials), even at world == 1 (NCCL test)
  int64_t row0, row1;     // global rows [row0, row1) are local
  double* halo;           // CSR: X rows [halo_lo, row0) then [row1, halo_hi) gathered from other ranks
  int64_t halo_lo;
  double *ag_send, *ag_all;    // alpha/g dd vectors: local (4k) / all ranks in rank order (world x 4k)
  double* mg_all;              // [M2 | G2 | rr2] of all ranks (world x (2k^2 + k))
  double *nrm_send, *nrm_all;  // column sums of x~^2: local (k) / all ranks (world x k)
  long long* tlog;   // optional clock64() phase log of the k x k kernels (REFINE_KXK_TIMING=1)
  // Rayleigh-Ritz preprocessing (Sec. 3.4): ritz values (k, descending), a zero k-vector (pass B
  // with D = 0 gives [X^T W | X^T X]), and the top-zero flag of the sweep that follows RR
  double *ritz, *zerod;
  int32_t top_zero;
  int32_t kjudge;    // > 0: ||E_L||_F over the leading kjudge columns (K > k)
  int32_t want_gram; // 1: kxk_finish reports max |X^T X - I| of the sweep's input in stats[6] (else -1)
  int* gate;         // refine_run reorthogonalisation gate: ST_OK when the gated pipeline must run
  int32_t normalize; // opts.normalize: kxk_finish folds 1/||x~_j|| into the top rows, Csig and scal
  int32_t kxk_h;     // 1: kxk_lu precomputes H1..H4 (scratch + 16 k^2 ..) for the clustered kxk_finish
  double* bdiag;     // tcgen05 pass B: FP64 partials of diag(X_2^T R_2), diag(X_2^T X_2) (n_chunk x 2 kp)
  int32_t fk_nobulk; // 1: kxk_finish's products stage with cp.async instead of bulk copies (REFINE_FK_BULK=0)
};

// X row of global index col: local rows first, else the halo (CSR row partition)
RF_DEV const double* xrow(const Ws& ws, const double* Xloc, int64_t col, int k) {
  if (ws.halo == nullptr || (col >= ws.row0 && col < ws.row1)) return Xloc + (col - ws.row0) * k;
  const int64_t h = (col < ws.row0) ? col - ws.halo_lo : (ws.row0 - ws.halo_lo) + (col - ws.row1);
  return ws.halo + h * k;
}

#define RF_TSTAMP(ws, i)                                                   \
  do {                                                                     \
    if ((ws).tlog && threadIdx.x == 0) (ws).tlog[i] = clock64();          \
  } while (0)

}  // namespace rf
