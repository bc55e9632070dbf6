// tc_passes.cuh -- NEXT-2: the tall-skinny products of the sweep on the 5th-generation
// tensor cores (tcgen05 / TMEM), in mixed precision ("some matrix-matrix
// multiplications in the applications of H and H^T may be computed in lower precision while keeping
// the accumulation and the small k x k computations in double").
//
// Precision scheme: every FP64 operand value v is rounded to f = fp32(v) and
// split f = v_hi + v_lo with v_hi = bf16(f), v_lo = bf16(f - v_hi) (the remainder is exact in
// FP32); a product a b is taken as
// a_hi b_hi + a_hi b_lo + a_lo b_hi on tcgen05.mma kind::f16 (bf16 x bf16 products are exact in the
// FP32 accumulator), which drops a_lo b_lo and the bf16 rounding of v_lo: relative error ~2^-16
// per product.  The FP32 TMEM accumulator sums at most KC = 512 rows before it is drained into FP64
// partials, and the partials are summed in FP64 (fixed order) -- so the k x k results carry a
// relative error ~1e-5 of sum |a||b|, i.e. the correction E_L is computed to ~1e-5 relative while
// the residual R = W - X D and every k x k step stay FP64: the refinement contracts at
// max(gamma, ~1e-5) per sweep and still reaches FP64 accuracy (tests/test_gpu_mixed.py).
//
// UMMA operand layout: canonical K-major, no swizzle: element (row r, k) of a tile at byte
// (r / 8) * SBO + (k / 8) * 128 + (r % 8) * 16 + (k % 8) * 2, LBO = 128 B (core matrices along K),
// SBO = (TK / 8) * 128 B (along M / N); descriptor version 1 (verified by tools/umma_test.cu).
#pragma once
#include <cuda_bf16.h>
#include "common.cuh"

namespace rf {

// ---------------------------------------------------------------- tcgen05 helpers
RF_DEV uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;              // descriptor version 1 (sm_100); base offset 0; SWIZZLE_NONE
  return d;
}
__host__ __device__ constexpr uint32_t umma_idesc_bf16(int m, int n) {   // BF16 x BF16 -> F32, K-major
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}
RF_DEV void umma_bf16(uint32_t tmem, uint64_t da, uint64_t db, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate));
}
RF_DEV void umma_commit(uint64_t* mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(mbar))
               : "memory");
}
RF_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
RF_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
// 16 consecutive FP32 accumulator columns of this warp's 32 TMEM lanes
RF_DEV void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(r[j]);
}
RF_DEV void tmem_ld8(uint32_t taddr, float (&v)[8]) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int j = 0; j < 8; ++j) v[j] = __uint_as_float(r[j]);
}
RF_DEV void tmem_st16(uint32_t taddr, const float (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n" ::"r"(
          taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])),
      "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])),
      "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
      "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])), "r"(__float_as_uint(v[15]))
      : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
}
// Two values v0, v1 (consecutive K) -> packed bf16x2 hi and lo words: v ~ f = fp32(v) (relative
// 2^-24), hi = bf16(f), lo = bf16(f - hi) (f - hi exact in FP32); lower half = v0.  One F2F per
// value; the bf16 rounding is the paired cvt.rn.bf16x2.f32.
RF_DEV void split2_bf16(double v0, double v1, uint32_t& hi, uint32_t& lo) {
  const float f0 = (float)v0, f1 = (float)v1;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(hi) : "f"(f1), "f"(f0));
  const float h0 = __uint_as_float(hi << 16), h1 = __uint_as_float(hi & 0xFFFF0000u);
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(lo) : "f"(f1 - h1), "f"(f0 - h0));
}
RF_DEV constexpr uint32_t kmaj_off(int r, int k, uint32_t sbo) {
  return (uint32_t)(r / 8) * sbo + (uint32_t)(k / 8) * 128u + (uint32_t)(r % 8) * 16u + (uint32_t)(k % 8) * 2u;
}

// ---------------------------------------------------------------- pass B on tcgen05 (k = 32 .. 128)
// [M2 | G2] = X_2^T [R_2 | X_2] over rows >= top (R = W - X D formed in FP64, rr_j = sum r_ij^2 in
// FP64), per CTA a contiguous row chunk; the CTA's FP64 partial goes to the passB2 slot layout
// (bpart[(c * NT + tile) * KP * 64 + a * 64 + b % 64] with [R | X] column b, X at KP, NT = 2 KP / 64;
// brr[c * KP + j]) so passB2_reduce_kernel<KP> sums the CTAs in fixed order.  k % 16 == 0, k >= 32:
// M = 128 (A = X^T, rows >= k zero), N = 2k.  One CTA per SM, warp-specialised:
//   warp 8 (producer): bulk-copies the X and W rows of each 16-row stage (contiguous 16 KB each,
//     cp.async.bulk completing on the slot's "full" mbarrier) into an NS-slot FP64 ring as soon as
//     the converters release a slot ("empty" mbarrier): up to (NS - 1) x 32 KB in flight per SM;
//   warps 0-7 (converters): form R = W - X D and the bf16 hi/lo splits of X and R into the UMMA
//     operand buffer of the stage; thread 0 issues tcgen05.mma (M = 128, N = 256, K = 16) for
//     hi*hi, hi*lo, lo*hi into the TMEM accumulator and commits to the buffer's mbarrier;
//   warps 9-12 (drain): every KC rows the tensor-core accumulator (TMEM columns 0-255) is added
//     into a second FP32 sum (TMEM columns 256-511) with round-to-nearest CUDA-core adds (error
//     control, header) and released for the next block; at the end the second sum is written to
//     the CTA's FP64 partial.
constexpr int TCB_K = 128, TCB_N = 256, TCB_NO = 2, TCB_CONV = 256;
constexpr int TCB_THREADS = TCB_CONV + 32 + 128 + 32;   // converters, producer, drain, MMA issue
constexpr int TCB_KC = 512;   // rows per TMEM block (tools/tcb_test.cu: 2048 -> 512 cuts the G error 2.6x, +1.6% time)
// Per padded width KP: TK rows per stage (a 16 KB FP64 slab of X, and one of W, at every KP), NS
// ring slots, the UMMA operand buffer (A = X^T padded to M = 128 rows, B = [R | X] with N = 2k rows).
template <int KP>
struct TcbCfg {
  static constexpr int TK = 16 * 128 / KP;                         // 16 / 32 / 64 rows
  static constexpr int NS = KP == 32 ? 4 : 5;
  static constexpr int SPB = TCB_KC / TK;                          // stages per accumulator block
  static constexpr uint32_t SBO = (TK / 8) * 128;
  static constexpr uint32_t A_BYTES = TCB_K * TK * 2, B_BYTES = 2 * KP * TK * 2;
  static constexpr uint32_t OPS = 2 * A_BYTES + 2 * B_BYTES;       // A_hi, A_lo, B_hi, B_lo
  static constexpr uint32_t ROWB = TK * KP * 8;                    // 16 KB
  static constexpr int SMEM = NS * 2 * ROWB + TCB_NO * OPS;        // 208 / 224 / 224 KB
  static constexpr int CB = KP / 16, QG = 8 / CB;                  // converter column blocks, quad groups
};

RF_DEV void conv_sync() { asm volatile("bar.sync 1, %0;\n" ::"n"(TCB_CONV) : "memory"); }

template <int KP>
__global__ void __launch_bounds__(TCB_THREADS, 1) passB_tc_kernel(Ws ws, const double* __restrict__ X) {
  using C = TcbCfg<KP>;
  constexpr int TK = C::TK, NS = C::NS;
  extern __shared__ __align__(16) unsigned char tcb_smem[];
  __shared__ __align__(8) uint64_t full[NS], empty[NS], mmad[TCB_NO], conv[TCB_NO], accf[2], acce[2];
  __shared__ uint32_t tmem_base;
  __shared__ double sd[KP];
  griddep_wait();   // (programmatic dependent launch: the predecessor's writes are visible after this)
  if (*ws.status != ST_OK) return;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t rows = ws.n_loc - ws.top;
  const int64_t per = ((rows + gridDim.x - 1) / gridDim.x + TK - 1) / TK * TK;
  const int64_t rb = ws.top + (int64_t)blockIdx.x * per;
  const int64_t re = (rb + per < ws.n_loc) ? rb + per : ws.n_loc;
  const int nst = (re > rb) ? (int)((re - rb + TK - 1) / TK) : 0;
  const int nblk = (nst + C::SPB - 1) / C::SPB;
  const int k = ws.k, N = 2 * k;                            // k % 16 == 0, KP / 2 < k <= KP
  unsigned char* F = tcb_smem;                              // [NS][X rows | W rows] FP64 (row stride k)
  unsigned char* OP = tcb_smem + NS * 2 * C::ROWB;          // [NO][A_hi | A_lo | B_hi | B_lo] bf16
  double* part = ws.bpart + (int64_t)blockIdx.x * 2 * KP * KP;   // passB2 slot layout (TA = KP, TB = 64)
  for (int j = tid; j < KP; j += TCB_THREADS) sd[j] = j < k ? ws.d[j] : 0.0;
  // A rows >= k (padding of M = 128) stay zero; the converters write rows < k only
  for (int e = tid; e < TCB_NO * (int)C::OPS / 16; e += TCB_THREADS) reinterpret_cast<uint4*>(OP)[e] = make_uint4(0, 0, 0, 0);
  fence_async_smem();
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base)),
                 "r"(2 * TCB_N));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], TCB_CONV / 32);
    }
    for (int i = 0; i < TCB_NO; ++i) {
      mbar_init(&mmad[i], 1);
      mbar_init(&conv[i], TCB_CONV);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&accf[i], 1);
      mbar_init(&acce[i], 4);
    }
  }
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base;
  double rr = 0.0, xr = 0.0, xx = 0.0;
  if (warp == TCB_CONV / 32) {                     // ---- producer
    if (lane == 0) {
      for (int t = 0; t < nst; ++t) {
        const int s = t % NS;
        if (t >= NS) {
          mbar_wait(&empty[s], ((t / NS) - 1) & 1);
          fence_async_smem();                       // converters' generic reads of slot s -> the refill
        }
        const int64_t r0 = rb + (int64_t)t * TK;
        const uint32_t bytes = (uint32_t)min((int64_t)TK, re - r0) * k * 8;
        unsigned char* f = F + s * 2 * C::ROWB;
        mbar_expect_tx(&full[s], 2 * bytes);
        bulk_g2s(f, X + r0 * k, bytes, &full[s]);
        bulk_g2s(f + C::ROWB, ws.W + r0 * k, bytes, &full[s]);
      }
    }
  } else if (warp == TCB_CONV / 32 + 5) {          // ---- MMA issue (one thread), decoupled from the converters
    if (lane == 0) {
      const uint32_t idesc = umma_idesc_bf16(TCB_K, 2 * ws.k);
      for (int t = 0; t < nst; ++t) {
        const int o = t % TCB_NO;
        mbar_wait(&conv[o], (t / TCB_NO) & 1);              // OP[o] written (and fenced) by every converter
        const int j = t / C::SPB, ts = t % C::SPB;          // accumulator block j, stage ts within it
        if (ts == 0 && j >= 1) mbar_wait(&acce[0], (j - 1) & 1);   // block j - 1 drained
        tc_fence_after();
        unsigned char* st = OP + o * C::OPS;
        const uint32_t a_hi = smem_u32(st), a_lo = smem_u32(st + C::A_BYTES), b_hi = smem_u32(st + 2 * C::A_BYTES),
                       b_lo = smem_u32(st + 2 * C::A_BYTES + C::B_BYTES);
#pragma unroll
        for (int kk = 0; kk < TK / 16; ++kk) {
          const uint32_t ko = kk * 256;                // 16 rows = 2 core matrices along K
          const uint64_t dah = umma_desc(a_hi + ko, 128, C::SBO), dal = umma_desc(a_lo + ko, 128, C::SBO);
          const uint64_t dbh = umma_desc(b_hi + ko, 128, C::SBO), dbl = umma_desc(b_lo + ko, 128, C::SBO);
          umma_bf16(tmem, dah, dbh, idesc, (ts > 0 || kk > 0) ? 1u : 0u);
          umma_bf16(tmem, dah, dbl, idesc, 1);
          umma_bf16(tmem, dal, dbh, idesc, 1);
        }
        umma_commit(&mmad[o]);
        if (ts == C::SPB - 1 || t == nst - 1) umma_commit(&accf[0]);
      }
    }
  } else if (warp > TCB_CONV / 32) {               // ---- drain: TMEM lanes 32 (warp % 4) ..
    const int m = 32 * (warp & 3) + lane;
    const uint32_t tl = tmem + ((uint32_t)(32 * (warp & 3)) << 16);
    for (int j = 0; j < nblk; ++j) {
      mbar_wait(&accf[0], j & 1);
      tc_fence_after();
#pragma unroll 1
      for (int c0 = 0; c0 < N; c0 += 16) {
        float v[16], u[16];
        tmem_ld16(tl + c0, v);
        if (j > 0) {
          tmem_ld16(tl + TCB_N + c0, u);
#pragma unroll
          for (int e = 0; e < 16; ++e) v[e] += u[e];
        }
        tmem_st16(tl + TCB_N + c0, v);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acce[0]);
    }
    if (nst == 0) {   // empty chunk: zero partial
      for (int e = tid - (TCB_CONV + 32); e < 2 * KP * KP; e += 128) part[e] = 0.0;
    } else {
      tc_fence_after();
#pragma unroll 1
      for (int c0 = 0; c0 < N; c0 += 16) {   // accumulator column c -> [R | X] column (X at KP)
        float v[16];
        tmem_ld16(tl + TCB_N + c0, v);
        const int pc = c0 < k ? c0 : KP + (c0 - k);
        double* p = part + ((pc >> 6) * KP + m) * 64 + (pc & 63);
        if (m < k) {
#pragma unroll
          for (int e = 0; e < 16; e += 2) *reinterpret_cast<double2*>(p + e) = make_double2(v[e], v[e + 1]);
        }
      }
    }
  } else {                                          // ---- converters
    // thread -> column col = 16 (w % CB) + (l & 15) and row quads q0, q0 + 2 QG, ... (q0 = (l >> 4) +
    // 2 (w / CB)): per warp instruction the FP64 reads are two 128 B row segments and the 8 B
    // operand stores two 128 B core-matrix rows (no bank conflicts)
    const int col = 16 * (warp % C::CB) + (lane & 15), q0 = (lane >> 4) + 2 * (warp / C::CB);
    const bool act = col < k;
    const double dcol = sd[col];
    for (int t = 0; t < nst; ++t) {
      const int s = t % NS, o = t % TCB_NO;
      mbar_wait(&full[s], (t / NS) & 1);                                 // rows landed
      if (t >= TCB_NO) mbar_wait(&mmad[o], ((t / TCB_NO) - 1) & 1);     // OP[o] free
      const int nr = (int)min((int64_t)TK, re - (rb + (int64_t)t * TK));
      const double* fx = reinterpret_cast<const double*>(F + s * 2 * C::ROWB);
      const double* fw = reinterpret_cast<const double*>(F + s * 2 * C::ROWB + C::ROWB);
      unsigned char* st = OP + o * C::OPS;
      unsigned char *Ahi = st, *Alo = st + C::A_BYTES, *Bhi = st + 2 * C::A_BYTES,
                    *Blo = st + 2 * C::A_BYTES + C::B_BYTES;
#pragma unroll
      for (int q = q0; q < (act ? TK / 4 : 0); q += 2 * C::QG) {
        const int r = 4 * q;
        double x[4], qv[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const bool v = r + j < nr;
          x[j] = v ? fx[(r + j) * k + col] : 0.0;
          const double w = v ? fw[(r + j) * k + col] : 0.0;
          qv[j] = __fma_rn(-x[j], dcol, w);             // R = W - X D (FP64)
          rr = __fma_rn(qv[j], qv[j], rr);
          xr = __fma_rn(x[j], qv[j], xr);               // diagonals of M2, G2 in FP64
          xx = __fma_rn(x[j], x[j], xx);
        }
        uint2 xh, xl, rh, rl;
        split2_bf16(x[0], x[1], xh.x, xl.x);
        split2_bf16(x[2], x[3], xh.y, xl.y);
        split2_bf16(qv[0], qv[1], rh.x, rl.x);
        split2_bf16(qv[2], qv[3], rh.y, rl.y);
        const uint32_t oa = kmaj_off(col, r, C::SBO);              // A = X^T: (m = col, k = row); B rows 0.. = R
        const uint32_t ob = kmaj_off(k + col, r, C::SBO);          // B rows k.. = X
        *reinterpret_cast<uint2*>(Ahi + oa) = xh;
        *reinterpret_cast<uint2*>(Alo + oa) = xl;
        *reinterpret_cast<uint2*>(Bhi + oa) = rh;
        *reinterpret_cast<uint2*>(Blo + oa) = rl;
        *reinterpret_cast<uint2*>(Bhi + ob) = xh;
        *reinterpret_cast<uint2*>(Blo + ob) = xl;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);        // this warp is done reading F[s]
      fence_async_smem();                           // operand stores -> the tensor core's async proxy
      mbar_arrive(&conv[o]);
    }
  }
  __syncthreads();
  double* srr = reinterpret_cast<double*>(tcb_smem);     // the FP64 ring is free now
  if (tid < TCB_CONV) {
    srr[tid] = rr;
    srr[TCB_CONV + tid] = xr;
    srr[2 * TCB_CONV + tid] = xx;
  }
  __syncthreads();
  if (tid < k) {   // column j: warps (j / 16) + CB g (g < QG), lanes (j % 16) and (j % 16) + 16, fixed order
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    for (int g = 0; g < C::QG; ++g) {
      const int t0 = 32 * ((tid >> 4) + C::CB * g) + (tid & 15);
      a0 += srr[t0] + srr[t0 + 16];
      a1 += srr[TCB_CONV + t0] + srr[TCB_CONV + t0 + 16];
      a2 += srr[2 * TCB_CONV + t0] + srr[2 * TCB_CONV + t0 + 16];
    }
    ws.brr[(int64_t)blockIdx.x * KP + tid] = a0;
    double* bd = ws.bdiag + (int64_t)blockIdx.x * 2 * KP;
    bd[tid] = a1;
    bd[KP + tid] = a2;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(2 * TCB_N));
}

// ---------------------------------------------------------------- pass C on tcgen05 (k = 32 .. 128)
// x~_i = w_i (Sigma D^-1) - x_i Csig for rows i >= top (eq. update-X through the implicit H, see
// passC_kernel), with the product x_i Csig -- an O(residual) term, PAPER.md:504-507 -- on tcgen05
// in the bf16x3 scheme and the w_i scaling, the subtraction and the column sums of squares in FP64.
// Transposed product per 64-column MMA: D (128 x 64, TMEM lanes = output columns, TMEM columns =
// slab rows) = A . B^T with K = 128.  k <= 64 packs G = 128 / KP row groups into one MMA: B row n =
// [x_{n} | x_{64 + n} | ...] (each KP wide, zero padded) and A = blockdiag(Csig^T, ..., Csig^T),
// so TMEM lane quarter g * KP / 32 .. holds the products of rows g * 64 + n (all 4 lane quarters
// and all epilogue warps stay busy at every k).  The M = 128 MMAs are bound by the SMEM read of A
// (tools/umma_sw_test.cu: ~48 cycles per MMA at N <= 64), so a slab is 64 G rows (64 KB of X).
// Operands use the 128-byte-swizzled K-major layout (row-contiguous 4-byte stores conflict-free).
// One CTA per SM, a contiguous row chunk per CTA, warp-specialised:
//   warp 12 (producer): one bulk copy per slab (contiguous X rows) into a 2-slot FP64 ring;
//   warps 0-3 (converters): bf16 hi/lo splits of the slab into the UMMA B buffer; thread 0
//     issues 3 x 8 tcgen05.mma (M = 128, N = 64, K = 16) into the slab's TMEM columns;
//   warps 4-11 (epilogue, TMEM lane quarter = warp % 4, 32 columns each): the W entries are loaded
//     (coalesced) before waiting for the MMA; tcgen05.ld, x~ = fma(w, s_j, -D), coalesced
//     stores of X~, FP64 column sums of squares.
constexpr int TCC_K = 128, TCC_NS = 2, TCC_TN = 64, TCC_NT = 4, TCC_RPW = 32;
constexpr int TCC_CONV = 128, TCC_EPI = 256, TCC_THREADS = TCC_CONV + TCC_EPI + 32;
constexpr uint32_t TCC_A_BYTES = TCC_K * TCC_K * 2, TCC_B_BYTES = TCC_TN * TCC_K * 2;
template <int KP>
struct TccCfg {
  static constexpr int G = 128 / KP;                               // row groups packed along K
  static constexpr int SROWS = TCC_TN * G;                         // slab rows: 64 / 128 / 256
  static constexpr uint32_t SLOT = SROWS * KP * 8;                 // 64 KB of X rows
  static constexpr int SMEM = 1024 + 2 * TCC_A_BYTES + 2 * TCC_B_BYTES + TCC_NS * SLOT;   // 225 KB
};

// 128-byte swizzle, K-major: element (r, k) of an R-row bf16 operand (64-wide K atoms, 8-row groups
// 1024 B apart, the 16-byte chunk index XOR row % 8); atoms 1024-byte aligned
RF_DEV constexpr uint32_t sw128_off(int r, int k, int R) {
  return (uint32_t)(k / 64) * (R * 128) + (uint32_t)(r / 8) * 1024 + (uint32_t)(r % 8) * 128 +
         (uint32_t)((((k % 64) / 8) ^ (r % 8)) * 16) + (uint32_t)(k % 8) * 2;
}
RF_DEV uint64_t umma_desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;                  // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;        // SBO: 8-row groups 1024 B apart
  d |= (uint64_t)1 << 46;                  // descriptor version 1
  d |= (uint64_t)2 << 61;                  // SWIZZLE_128B
  return d;
}
// K step kk (16 elements) of an R-row swizzled operand at base: the start moves 32 B inside the atom
RF_DEV uint64_t sw128_kdesc(uint32_t base, int kk, int R) {
  return umma_desc_sw128(base + (uint32_t)(kk / 4) * (R * 128) + (uint32_t)(kk % 4) * 32);
}
RF_DEV void conv_sync_c() { asm volatile("bar.sync 1, %0;\n" ::"n"(TCC_CONV) : "memory"); }

template <int KP>
__global__ void __launch_bounds__(TCC_THREADS, 1) passC_tc_kernel(Ws ws, const double* X, double* out) {
  using C = TccCfg<KP>;
  constexpr int G = C::G, SROWS = C::SROWS;
  extern __shared__ __align__(16) unsigned char tcc_raw[];
  __shared__ __align__(8) uint64_t full[TCC_NS], empty[TCC_NS], opfree, accf[TCC_NT], acce[TCC_NT];
  __shared__ uint32_t tmem_base;
  __shared__ double ssc[KP];
  griddep_wait();   // (programmatic dependent launch: the predecessor's writes are visible after this)
  if (*ws.status != ST_OK) return;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int k = ws.k;                                // k % 16 == 0, KP / 2 < k <= KP
  const int64_t rows = ws.n_loc - ws.top;
  const int64_t per = ((rows + gridDim.x - 1) / gridDim.x + SROWS - 1) / SROWS * SROWS;
  const int64_t rb = ws.top + (int64_t)blockIdx.x * per;
  const int64_t re = (rb + per < ws.n_loc) ? rb + per : ws.n_loc;
  const int nst = (re > rb) ? (int)((re - rb + SROWS - 1) / SROWS) : 0;
  unsigned char* base = tcc_raw + ((1024 - (smem_u32(tcc_raw) & 1023)) & 1023);   // 1024-B aligned
  unsigned char* Ahi = base;
  unsigned char* Alo = base + TCC_A_BYTES;
  unsigned char* Bhi = base + 2 * TCC_A_BYTES;
  unsigned char* Blo = Bhi + TCC_B_BYTES;
  unsigned char* F = Blo + TCC_B_BYTES;                              // [NS][slab rows] FP64 (row stride k)
  // A = blockdiag(Csig^T): element (m = g KP + j, l = g KP + l') = Csig[l'][j] (ld k), split once
  for (int e = tid; e < TCC_K * TCC_K / 2; e += TCC_THREADS) {
    const int m = e % TCC_K, l = 2 * (e / TCC_K);
    const int j = m % KP, lp = l % KP;
    const bool ok = (m / KP == l / KP) && j < k && lp < k;
    uint32_t hi, lo;
    split2_bf16(ok ? ws.Csig[lp * k + j] : 0.0, ok ? ws.Csig[(lp + 1) * k + j] : 0.0, hi, lo);
    const uint32_t off = sw128_off(m, l, TCC_K);
    *reinterpret_cast<uint32_t*>(Ahi + off) = hi;
    *reinterpret_cast<uint32_t*>(Alo + off) = lo;
  }
  for (int j = tid; j < KP; j += TCC_THREADS) ssc[j] = j < k ? ws.scal[j] : 0.0;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base)),
                 "r"(TCC_NT * TCC_TN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    for (int i = 0; i < TCC_NS; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], TCC_CONV / 32);
    }
    mbar_init(&opfree, 1);
    for (int i = 0; i < TCC_NT; ++i) {
      mbar_init(&accf[i], 1);
      mbar_init(&acce[i], TCC_EPI / 32);
    }
  }
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base;
  double nacc = 0.0;
  if (warp == (TCC_CONV + TCC_EPI) / 32) {          // ---- producer
    if (lane == 0) {
      for (int t = 0; t < nst; ++t) {
        const int s = t % TCC_NS;
        if (t >= TCC_NS) {
          mbar_wait(&empty[s], ((t / TCC_NS) - 1) & 1);
          fence_async_smem();                       // converters' generic reads of slot s -> the refill
        }
        const int64_t r0 = rb + (int64_t)t * SROWS;
        const uint32_t bytes = (uint32_t)min((int64_t)SROWS, re - r0) * k * 8;
        mbar_expect_tx(&full[s], bytes);
        bulk_g2s(F + s * C::SLOT, X + r0 * k, bytes, &full[s]);
      }
    }
  } else if (warp < TCC_CONV / 32) {                // ---- converters + MMA issue
    const uint32_t idesc = umma_idesc_bf16(TCC_K, TCC_TN);
    for (int t = 0; t < nst; ++t) {
      const int s = t % TCC_NS;
      mbar_wait(&full[s], (t / TCC_NS) & 1);
      if (t >= 1) mbar_wait(&opfree, (t - 1) & 1);   // the previous slab's MMAs have read B
      const int nr = (int)min((int64_t)SROWS, re - (rb + (int64_t)t * SROWS));
      const double* fx = reinterpret_cast<const double*>(F + s * C::SLOT);
      // warp w: slab rows w, w + 4, ... (row r -> B row r % 64, K columns (r / 64) KP + l');
      // lane: l' = 2 lane (+ 64 for KP = 128)
#pragma unroll 4
      for (int r = warp; r < SROWS; r += TCC_CONV / 32) {
        const int n = r % TCC_TN, g = r / TCC_TN;
#pragma unroll
        for (int h = 0; h < (KP + 63) / 64; ++h) {
          const int lp = 64 * h + 2 * lane;
          if (lp < KP) {
            double2 v = make_double2(0.0, 0.0);
            if (r < nr && lp < k) v = *reinterpret_cast<const double2*>(fx + r * k + lp);
            uint32_t hi, lo;
            split2_bf16(v.x, v.y, hi, lo);
            const uint32_t off = sw128_off(n, g * KP + lp, TCC_TN);
            *reinterpret_cast<uint32_t*>(Bhi + off) = hi;
            *reinterpret_cast<uint32_t*>(Blo + off) = lo;
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);        // X rows of the slab consumed
      fence_async_smem();
      tc_fence_before();
      conv_sync_c();
      if (tid == 0) {
        const int a = t % TCC_NT;
        if (t >= TCC_NT) mbar_wait(&acce[a], ((t / TCC_NT) - 1) & 1);   // TMEM columns read out
        tc_fence_after();
        const uint32_t td = tmem + (uint32_t)(a * TCC_TN);
        const uint32_t ah = smem_u32(Ahi), al = smem_u32(Alo), bh = smem_u32(Bhi), bl = smem_u32(Blo);
#pragma unroll
        for (int kk = 0; kk < TCC_K / 16; ++kk) {
          const uint64_t dah = sw128_kdesc(ah, kk, TCC_K), dal = sw128_kdesc(al, kk, TCC_K);
          const uint64_t dbh = sw128_kdesc(bh, kk, TCC_TN), dbl = sw128_kdesc(bl, kk, TCC_TN);
          umma_bf16(td, dah, dbh, idesc, kk > 0);
          umma_bf16(td, dah, dbl, idesc, 1);
          umma_bf16(td, dal, dbh, idesc, 1);
        }
        umma_commit(&opfree);
        umma_commit(&accf[a]);
      }
    }
  } else {                                          // ---- epilogue: TMEM lane m = 32 (warp % 4) + lane
    const int m = 32 * (warp & 3) + lane, g = m / KP, j = m % KP;
    const int rh = (warp - TCC_CONV / 32) / 4 * TCC_RPW;
    const bool act = j < k;
    const double sj = ssc[j];
    const uint32_t tl = tmem + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)rh;
    for (int t = 0; t < nst; ++t) {
      const int a = t % TCC_NT;
      const int64_t r0 = rb + (int64_t)t * SROWS + g * TCC_TN + rh;   // slab rows of TMEM columns rh ..
      const int nr = (int)min((int64_t)TCC_RPW, re - r0);
      double w[TCC_RPW];
#pragma unroll
      for (int r = 0; r < TCC_RPW; ++r) w[r] = (act && r < nr) ? __ldcs(ws.W + (r0 + r) * k + j) : 0.0;
      mbar_wait(&accf[a], (t / TCC_NT) & 1);
      tc_fence_after();
      float v[TCC_RPW];
#pragma unroll
      for (int c = 0; c < TCC_RPW; c += 16) tmem_ld16(tl + (uint32_t)(a * TCC_TN + c), *reinterpret_cast<float(*)[16]>(v + c));
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acce[a]);
#pragma unroll
      for (int r = 0; r < TCC_RPW; ++r) {
        if (act && r < nr) {
          const double x = __fma_rn(w[r], sj, -(double)v[r]);
          __stcs(out + (r0 + r) * k + j, x);
          nacc = __fma_rn(x, x, nacc);
        }
      }
    }
  }
  __syncthreads();
  double* snorm = reinterpret_cast<double*>(F);      // the ring is free now
  if (warp >= TCC_CONV / 32 && warp < (TCC_CONV + TCC_EPI) / 32) snorm[tid - TCC_CONV] = nacc;
  __syncthreads();
  if (tid < k) {   // column j: lanes m = g KP + j of both row halves, groups and halves in fixed order
    double v = 0.0;
    for (int g = 0; g < G; ++g)
#pragma unroll
      for (int h = 0; h < TCC_EPI / 128; ++h) v += snorm[128 * h + g * KP + tid];
    ws.nslot[(int64_t)blockIdx.x * KP + tid] = v;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(TCC_NT * TCC_TN));
}

}  // namespace rf
