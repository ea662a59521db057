// Fused dequantize-and-multiply GEMV for the Q-Palette palette on sm_100a.
//
// y[beta][row] = s[row] * sum_k W_hat[row][k] * x'[beta][k],  batch <= 8
//
// Design:
//  * persistent grid, one CTA per SM, 16 warps (12 above 4 bits/weight); a replicated decode
//    table in shared memory (entries x 32 replicas, bank = lane: 128 KB for TCQ tb = 9);
//    the RT x KT tiles (32 rows x 256 cols, LAYOUT.md) are split into contiguous, k-minor
//    ranges per CTA and per warp (flat stream-K: balanced to within one tile). Work units are
//    single tiles, or row pairs (RP = 2: the two row tiles share the activation fragments) at
//    batch 8 with small tables;
//  * each lane owns one 256-weight trellis / code run per tile. A tile's codes are one
//    contiguous 512c-byte block; every warp streams its units into a private NS-stage ring in
//    shared memory with 1-D bulk-async copies (cp.async.bulk, the TMA engine; one elected lane
//    issues them, completion on a per-stage mbarrier) and refills a stage as soon as it is read
//    (ordered by a warp reduction over the loaded words), so code loads never block instruction
//    issue. Each lane reads its 4c stream words with c conflict-free 128-bit shared loads;
//  * decode per weight pair (TCQ): funnel-shift window -> IMAD hash (w+1)w -> IMAD key shift ->
//    LOP3 mask|lane -> one conflict-free LDS (bank = lane) -> half2; VQ/NUQ/UNIF: shift ->
//    LOP3 -> LDS. Pairs land directly in mma.sync m16n8k16 A-fragment registers (step j IS
//    fragment register j); the activations are the B fragment (batch in N <= 8; one 256-bit
//    load per lane per half tile, or shared memory with XM >= 1), fp32 accumulation;
//  * epilogue: per-row scales prefetched per row tile; owned row tiles stored directly; split
//    row tiles red.add into a pre-zeroed fp32 y, or (fp16 y / QP_DETERMINISTIC) warp partials ->
//    CTA shared-memory reduction -> in-order cross-CTA fixup;
//  * programmatic dependent launch: table build and the first code copies happen before
//    griddepcontrol.wait (they read only immutable layer data); dependents are triggered after
//    the main loop.
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <algorithm>
#include <utility>

#include "qp_internal.h"

namespace qp {

template <int... Is, class F>
__device__ __forceinline__ void static_for_impl(std::integer_sequence<int, Is...>, F&& f) {
  (f(std::integral_constant<int, Is>{}), ...);
}
template <int N, class F>
__device__ __forceinline__ void static_for(F&& f) {
  static_for_impl(std::make_integer_sequence<int, N>{}, f);
}

// Dynamic shared memory of the GEMV kernels; the decode table starts at byte 0. Referencing the
// symbol directly (rather than through a generic pointer) lets ptxas fold the table base into
// the LDS immediate, saving one IADD per decoded pair.
extern __shared__ __align__(1024) uint8_t qp_smem[];
// The shared::cta address of qp_smem: the first 1 KB of a CTA's shared window is reserved on
// sm_90+/sm_100, so dynamic shared memory (no static shared memory in these kernels) starts at
// 0x400. The kernel verifies this once at entry (trap otherwise) and the LDS below carries the
// base as an immediate, saving one IADD per decoded pair.
constexpr uint32_t kDynSmemBase = 0x400;
__device__ __forceinline__ uint32_t lds32(uint32_t off) {
  uint32_t v;
  asm volatile("ld.shared.b32 %0, [%1+1024];" : "=r"(v) : "r"(off));
  return v;
}

// Stream bits [O, O+NB) of a lane's circular MSB-first word stream w[0..NW), returned with
// the field's least significant bit at bit POS (other bits are garbage).
template <int O, int NB, int POS, int NW>
__device__ __forceinline__ uint32_t field(const uint32_t* w) {
  constexpr int E = O + NB - 1;
  constexpr int WO = (O >> 5) % NW;
  constexpr int WE = (E >> 5) % NW;
  constexpr int PL = 31 - (E & 31);
  constexpr int SH = PL - POS;
  if constexpr (WO == WE) {
    if constexpr (SH >= 0) return w[WE] >> SH;
    else return w[WE] << (-SH);
  } else {
    static_assert(SH > 0 && SH < 32, "spanning field");
    return __funnelshift_r(w[WE], w[WO], SH);
  }
}

// (a & MASK) | c as one LOP3 (ptxas otherwise re-masks c with a second LOP3 for some masks)
template <uint32_t MASK>
__device__ __forceinline__ uint32_t and_or(uint32_t a, uint32_t c) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(d) : "r"(a), "n"(MASK), "r"(c));
  return d;
}


// ---- mbarrier + 1-D bulk async copy (TMA engine) helpers ---------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n\tfence.proxy.async.shared::cta;" ::: "memory");
}
// arrive (count 1) and announce `bytes` of transaction for the current phase
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "QP_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra QP_WAIT_%=;\n}" :: "r"(bar), "r"(parity) : "memory");
}
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
// global -> shared bulk copy of `bytes` (multiple of 16, 16-B aligned), completing on `bar`;
// the codes are read exactly once: L2 evict-first.
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar, uint64_t pol) {
#ifdef QP_NO_EVICT_FIRST
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
  return;
#endif
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
      :: "r"(dst), "l"(src), "r"(bytes), "r"(bar), "l"(pol) : "memory");
}
// fire-and-forget fp32 add (RED, no return): atomicAdd with an unused result is not always lowered to
// RED -- in kernels that also contain system-scope fences ptxas keeps a returning ATOM. No "memory"
// clobber: the reductions are relaxed (ordered before the completion counter's acq_rel atomic, itself
// a volatile asm) and must not pin the surrounding loads / stores of the epilogue.
__device__ __forceinline__ void red_add_f32(float* p, float v) {
  asm volatile("red.relaxed.gpu.global.add.f32 [%0], %1;" :: "l"(p), "f"(v));
}
__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}

template <int REPS>
struct RepBits {
  static constexpr int value = REPS == 32 ? 7 : REPS == 16 ? 6 : REPS == 8 ? 5 : REPS == 4 ? 4 : REPS == 2 ? 3 : 2;
};

// One decoded weight pair (half2 bits, low half = even column) of step J.
template <int MODE, int C, int L, int TB, int REPS>
struct Dec {
  static constexpr int NW = 4 * C;
  static constexpr int PB = RepBits<REPS>::value;   // log2(REPS * 4): key -> byte offset shift
  // key shift of the TCQ modes: the (sign, idx) key sits at bits [L-1-TB, L-1] of p and must land
  // at bit PB of the table byte offset
  static constexpr int KSH = PB - (L - 1 - TB);
  template <int J>
  __device__ __forceinline__ static uint32_t step(const uint32_t* w, uint32_t laneoff, uint32_t mulk) {
    if constexpr (MODE == DEC_TCQ_PRESIGNED) {
      // window int(r[J*s : J*s+L]) -> p = (w+1) w mod 2^L -> key = bits
      // [L-1-TB, L-1] of p (sign bit on top) -> pre-signed entry.
      // The key shift is a multiply by mulk = 2^KSH held in a register (a runtime value to ptxas),
      // so it issues as a second IMAD on the FMA pipe instead of an IADD3/SHF on the ALU pipe,
      // which the window funnel shift and the mask already load (2 ALU + 2 FMA ops per pair).
      const uint32_t win = field<J * C, L, 0, NW>(w);
      const uint32_t p = win * win + win;
      constexpr uint32_t MASK = ((1u << (TB + 1)) - 1u) << PB;
      const uint32_t k = KSH >= 0 ? p * mulk : (p >> (KSH < 0 ? -KSH : 0));
      return lds32(and_or<MASK>(k, laneoff));
    } else if constexpr (MODE == DEC_TCQ_UNSIGNED) {
      const uint32_t win = field<J * C, L, 0, NW>(w);
      const uint32_t p = win * win + win;
      constexpr uint32_t MASK = ((1u << TB) - 1u) << PB;
      const uint32_t k = KSH >= 0 ? p * mulk : (p >> (KSH < 0 ? -KSH : 0));
      const uint32_t v = lds32(((k & MASK) | laneoff));
      return v ^ ((p << (16 - L)) & 0x8000u);             // sflp on the first coordinate
    } else if constexpr (MODE == DEC_LUT2) {
      const uint32_t f = field<J * C, C, PB, NW>(w);
      return lds32(((f & (((1u << C) - 1u) << PB)) | laneoff));
    } else {  // DEC_SCALAR: C = 2 * TB, even-column code first
      const uint32_t f0 = field<J * C, TB, PB, NW>(w);
      const uint32_t f1 = field<J * C + TB, TB, PB, NW>(w);
      constexpr uint32_t MASK = ((1u << TB) - 1u) << PB;
      const uint32_t h0 = lds32(((f0 & MASK) | laneoff));
      const uint32_t h1 = lds32(((f1 & MASK) | laneoff));
      return __byte_perm(h0, h1, 0x5410);
    }
  }
};

__device__ __forceinline__ void mma16816(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// 8 regs = 16 halves = one full 32-byte sector per lane: a single 256-bit load on sm_100
// (LDG.E.ENL2.256); two 128-bit loads would each touch 32 half-used sectors per warp at batch 8
// (8 rows x 4 column groups), doubling the L1 tag / sector work that throttles the MIO queue.
__device__ __forceinline__ void load_x8(uint32_t* dst, const __half* src) {
#ifdef QP_X_LDG128
  const uint4 v0 = __ldg(reinterpret_cast<const uint4*>(src));
  const uint4 v1 = __ldg(reinterpret_cast<const uint4*>(src) + 1);
  dst[0] = v0.x; dst[1] = v0.y; dst[2] = v0.z; dst[3] = v0.w;
  dst[4] = v1.x; dst[5] = v1.y; dst[6] = v1.z; dst[7] = v1.w;
#else
  asm volatile("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(dst[0]), "=r"(dst[1]), "=r"(dst[2]), "=r"(dst[3]), "=r"(dst[4]), "=r"(dst[5]), "=r"(dst[6]),
                 "=r"(dst[7])
               : "l"(src));
#endif
}

// Decode one tile's 128 steps of this lane and multiply-accumulate (GEMV) or store (dequant).
// x' B fragments: xb[0..15] (kappa 0..7) and xb[16..31] (kappa 8..15). The second half of this
// tile's activations (x_hi) is loaded when the tile starts and the first half of the next tile's
// (x_next) once kappa 0..7 are done, so activation loads never sit on the critical path and
// need no extra registers. Lanes with no batch row (x_hi == nullptr) keep zeros (loading a valid
// row for them instead measured 10-25% slower: profiles/r1/ab_xs_r1.md section 4).
__device__ __forceinline__ uint2 lds64(uint32_t addr) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(addr));
  return v;
}

// 256-bit activation load through L1 (for x' written by the same launch, e.g. the multi-layer
// engine's in-kernel rotation: no .nc path)
__device__ __forceinline__ void load_x8_coh(uint32_t* dst, const __half* src) {
#ifdef QP_ENG_NC_X
  asm volatile("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(dst[0]), "=r"(dst[1]), "=r"(dst[2]), "=r"(dst[3]), "=r"(dst[4]), "=r"(dst[5]), "=r"(dst[6]),
                 "=r"(dst[7])
               : "l"(src)
               : "memory");
  return;
#endif
  asm volatile("ld.global.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(dst[0]), "=r"(dst[1]), "=r"(dst[2]), "=r"(dst[3]), "=r"(dst[4]), "=r"(dst[5]), "=r"(dst[6]),
                 "=r"(dst[7])
               : "l"(src)
               : "memory");
}

template <int MODE, int C, int L, int TB, int REPS, bool DEQ, bool XS, bool COH = false>
__device__ __forceinline__ void tile_body(const uint32_t* w, uint32_t laneoff, uint32_t mulk, uint32_t* xb,
                                          float (&acc)[2][4],
                                          uint32_t* wout_lane, int ldw_words, const __half* x_hi,
                                          const __half* x_next, uint32_t xs_addr) {
  using D = Dec<MODE, C, L, TB, REPS>;
  if constexpr (!DEQ && XS) {
    const uint2 bx = lds64(xs_addr);
    xb[0] = bx.x;
    xb[1] = bx.y;
  }
  if constexpr (!DEQ && !XS) {
    if (x_hi) {
      if constexpr (COH) {
        load_x8_coh(xb + 16, x_hi);
        load_x8_coh(xb + 24, x_hi + 16);
      } else {
        load_x8(xb + 16, x_hi);
        load_x8(xb + 24, x_hi + 16);
      }
    }
  }
  static_for<16>([&](auto KAP) {
    constexpr int kap = decltype(KAP)::value;
    static_for<2>([&](auto M) {
      constexpr int m = decltype(M)::value;
      constexpr int j = 8 * kap + 4 * m;
      const uint32_t a0 = D::template step<j + 0>(w, laneoff, mulk);
      const uint32_t a1 = D::template step<j + 1>(w, laneoff, mulk);
      const uint32_t a2 = D::template step<j + 2>(w, laneoff, mulk);
      const uint32_t a3 = D::template step<j + 3>(w, laneoff, mulk);
      if constexpr (DEQ) {
        // step -> (row, col): row = 16m + g + 8(rho&1), col = 64q + 4kap + 2(rho>>1)
        uint32_t* p = wout_lane + (16 * m) * ldw_words + 2 * kap;
        p[0] = a0;
        p[8 * ldw_words] = a1;
        p[1] = a2;
        p[8 * ldw_words + 1] = a3;
      } else if constexpr (XS) {
        // B fragment of k-step kap in xb[2(kap&1)..]; the next one is requested one k-step ahead
        if constexpr (m == 0 && kap + 1 < 16) {
          const uint2 bx = lds64(xs_addr + 8 * (kap + 1));
          xb[2 * ((kap + 1) & 1)] = bx.x;
          xb[2 * ((kap + 1) & 1) + 1] = bx.y;
        }
        mma16816(acc[m], a0, a1, a2, a3, xb[2 * (kap & 1)], xb[2 * (kap & 1) + 1]);
      } else {
        mma16816(acc[m], a0, a1, a2, a3, xb[2 * kap], xb[2 * kap + 1]);
      }
    });
    if constexpr (!DEQ && !XS && kap == 7) {
      if (x_next) {
        if constexpr (COH) {
          load_x8_coh(xb, x_next);
          load_x8_coh(xb + 8, x_next + 16);
        } else {
          load_x8(xb, x_next);
          load_x8(xb + 8, x_next + 16);
        }
      }
    }
  });
}

// Replicated decode table: entry e, replica r at byte e*REPS*4 + r*4 (bank = replica = lane mod
// REPS). Built straight from the compact global table in two phases so that the table loads can
// be issued before the first tile's code loads (they would otherwise queue behind ~40 KB per SM
// of HBM requests) and stored once they arrive: 16-byte chunk i holds 4 replicas of entry
// i / (REPS/4), so a warp writes 512 contiguous bytes per STS.128 (conflict-free) and the lanes
// that need the same entry word share one L1 request.
template <int REPS, int NT, int ENTRIES>
struct TableBuild {
  // the compact table has exactly ENTRIES words (the host pads it): no bounds predicates
  static constexpr int V4 = REPS / 4;
  static constexpr int TOTAL = ENTRIES * V4;             // 16-byte chunks of the image
  static constexpr int B = (TOTAL + NT - 1) / NT;        // chunks per thread
  static constexpr bool EXACT = TOTAL % NT == 0;
  uint32_t v[B];
  __device__ __forceinline__ void load(const uint32_t* __restrict__ g) {
#pragma unroll
    for (int k = 0; k < B; ++k) {
      const int i = threadIdx.x + k * NT;
      v[k] = (EXACT || k + 1 < B || i < TOTAL) ? __ldg(g + i / V4) : 0u;
    }
  }
  __device__ __forceinline__ void store(uint8_t* tab) const {
#pragma unroll
    for (int k = 0; k < B; ++k) {
      const int i = threadIdx.x + k * NT;
      if (EXACT || k + 1 < B || i < TOTAL) *reinterpret_cast<uint4*>(tab + (size_t)i * 16) = make_uint4(v[k], v[k], v[k], v[k]);
    }
  }
};

// Shared-memory plan of one kernel variant (compile-time part):
//   [0, TAB)                     replicated decode table (entries x REPS x 4 B)
//   [TAB, TAB + 1024)            one mbarrier per ring stage (<= 16 warps x 4 stages)
//   [XS_OFF, + xs_bytes)         x' of every batch row, padded layout (XS variants only)
//   [.., + NWARP * ns * STAGE)   per-warp code rings of ns stages, 512*CMAX bytes each
// The epilogue's warp partials alias [XS_OFF, ...) after the loop. ns and xs_bytes are chosen at
// launch (launch_plan) from the batch and d_in.
#ifndef QP_XS_WARPS
#define QP_XS_WARPS 16
#endif
template <int MODE, int CLO, int CHI, int TB, int REPS, bool XS = false>
struct Plan {
  static constexpr int CMAX = CLO > CHI ? CLO : CHI;
  static constexpr int ENTRIES = MODE == DEC_TCQ_PRESIGNED ? (2 << TB) : MODE == DEC_LUT2 ? (1 << CLO) : (1 << TB);
  static constexpr int TAB = ENTRIES * REPS * 4 < 4096 ? 4096 : ENTRIES * REPS * 4;
  static constexpr int SMEM_MAX = 232448;          // sm_100 opt-in per block
  static constexpr int STAGE = 512 * CMAX;
  // register budget (128 regs x 512 threads, no spills); x' in shared memory frees the 32
  // B-fragment registers (QP_XS_WARPS experiments with more warps)
#ifndef QP_WIDE_CMAX
#define QP_WIDE_CMAX 8   // 16 warps up to c = 8 (4 bits); 12 above (register budget)
#endif
  static constexpr int NWARP = CMAX <= QP_WIDE_CMAX ? (XS ? QP_XS_WARPS : 16) : 12;
  static constexpr int BAR_OFF = TAB;
  static constexpr int XS_OFF = TAB + 1024;
  static constexpr int PART = NWARP * 2 * 256 * 4;  // epilogue warp partials
  static constexpr int AVAIL = SMEM_MAX - XS_OFF;   // for x' + rings
  static_assert(AVAIL >= NWARP * STAGE && AVAIL >= PART, "shared-memory plan does not fit");
};

// x' staged in shared memory (XS): batch row g at g*RS, element k at (k/64)*136 + (k%64)*2 within
// the row, RS = 136*(d_in/64) rounded up to 32 (mod 128). A lane's B fragment for k-step kappa
// (4 consecutive elements 64q + 4kappa, LAYOUT.md section 2) is one 8-byte load; the 8-byte pad
// per 64-element group and RS = 32 (mod 128) put the 16 lanes of a half-warp (g < 4, q < 4) on
// 16 distinct bank pairs: conflict-free.
__host__ __device__ constexpr int xs_row_stride(int d_in) {
  const int base = (d_in / 64) * 136;
  return base + ((32 - base % 128) + 128) % 128;
}

__device__ __forceinline__ uint32_t owner_of(uint32_t t, uint32_t lo, uint32_t n, uint32_t parts) {
  // part p owns [lo + n*p/parts, lo + n*(p+1)/parts); returns the p that contains t
  return ((t - lo + 1) * parts - 1) / n;
}

__device__ __forceinline__ void store_out(const GemvParams& p, int rt, int row, int b, float v, float scale) {
  int i = 0;
#pragma unroll 1
  while (i + 1 < p.n_out && rt >= p.rt_begin[i + 1]) ++i;
  const int grow = (rt - p.rt_begin[i]) * kTileRows + row;
  v *= scale;
  if (p.n_peers > 0) {
    // fused all-gather: the final value goes straight into every rank's y_full over NVLink
    // (peer stores through the mapped pointers; rank-local for this rank)
    const size_t off = (size_t)b * p.peer_ld + p.peer_row0 + grow;
#pragma unroll 1
    for (int k = 0; k < p.n_peers; ++k) {
      if (p.y_f32) reinterpret_cast<float*>(p.peer_y[k])[off] = v;
      else reinterpret_cast<__half*>(p.peer_y[k])[off] = __float2half_rn(v);
    }
    return;
  }
  if (p.y_f32) {
    float* dst = reinterpret_cast<float*>(p.y[i]) + (size_t)b * p.ldy[i] + grow;
    *dst = p.y_accum ? *dst + v : v;        // the owning warp is the only writer of this element
  }
  else reinterpret_cast<__half*>(p.y[i])[(size_t)b * p.ldy[i] + grow] = __float2half_rn(v);
}

// Fused all-gather completion: after every CTA's stores, the grid's last CTA increments this
// rank's arrival flag on every peer (system scope); qp_peer_wait_kernel on each rank waits for
// all ranks' flags. Fence / relaxed-atomic / fence gives the release-acquire chain.
__device__ __forceinline__ void peer_signal(const GemvParams& p) {
  if (p.n_peers <= 0) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    if (atomicAdd(p.peer_counter, 1) == (int)gridDim.x - 1) {
      p.peer_counter[0] = 0;                      // self-reset for the next launch
      __threadfence_system();
      for (int k = 0; k < p.n_peers; ++k) atomicAdd_system(p.peer_flag[k] + p.peer_rank, 1u);
    }
  }
}



// ---- fused activation rotation (XM == 2) --------------------------------------------------
// x' = (1/sqrt(b)) blockdiag(H_b) D x computed by every CTA into its staged x'.
// The arithmetic is that of qp_rht_kernel<8> step for step (3 butterfly stages in registers,
// 5 across lanes, the rest through shared memory, fp32, one RNE rounding), so the result is
// bitwise the one the separate rotation kernel writes. A warp owns a 256-element segment; a round
// transforms NWARP / (b/256) blocks; the scratch holds one fp32 block per concurrently processed
// block (NWARP * 256 floats).
__host__ __device__ constexpr int rot_scratch_offset(int batch, int rs) { return ((batch * rs + 127) / 128) * 128; }

template <int NWARP>
__device__ __forceinline__ void rotate_x(const GemvParams& p, uint8_t* xs, float* scratch) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int bsz = p.rht_block, spb = bsz >> 8;          // 256-element segments per block
  const int bpr = NWARP / spb;                          // blocks per round
  const int nblk = p.d_in / bsz, total = p.batch * nblk;
  const int slot = warp / spb, seg = warp - slot * spb;
  const int e0 = seg * 256 + lane * 8;                  // first element of this lane in its block
  for (int r0 = 0; r0 < total; r0 += bpr) {
    const int gb = r0 + slot;
    const bool act = slot < bpr && gb < total;
    const int beta = act ? gb / nblk : 0, blk = act ? gb - beta * nblk : 0;
    float v[8];
    if (act) {
      const size_t base = (size_t)beta * p.d_in + (size_t)blk * bsz + e0;
      if (p.x_dtype == 0) {
        const uint4 u = __ldg(reinterpret_cast<const uint4*>(reinterpret_cast<const __half*>(p.x_raw) + base));
        const __half2* h = reinterpret_cast<const __half2*>(&u);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float2 f = __half22float2(h[k]);
          v[2 * k] = f.x;
          v[2 * k + 1] = f.y;
        }
      } else if (p.x_dtype == 1) {
        const __nv_bfloat16* xb16 = reinterpret_cast<const __nv_bfloat16*>(p.x_raw) + base;
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = __bfloat162float(xb16[i]);
      } else {
        const float4 f0 = __ldg(reinterpret_cast<const float4*>(reinterpret_cast<const float*>(p.x_raw) + base));
        const float4 f1 = __ldg(reinterpret_cast<const float4*>(reinterpret_cast<const float*>(p.x_raw) + base) + 1);
        v[0] = f0.x; v[1] = f0.y; v[2] = f0.z; v[3] = f0.w; v[4] = f1.x; v[5] = f1.y; v[6] = f1.z; v[7] = f1.w;
      }
      const int gi = blk * bsz + e0;                    // index within the row (8 | gi: one sign word)
      const uint32_t sw = __ldg(p.rht_signs + (gi >> 5)) >> (gi & 31);
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if ((sw >> i) & 1u) v[i] = -v[i];
#pragma unroll
      for (int h = 1; h < 8; h <<= 1)
#pragma unroll
        for (int i = 0; i < 8; ++i)
          if ((i & h) == 0) {
            const float a0 = v[i], a1 = v[i + h];
            v[i] = a0 + a1;
            v[i + h] = a0 - a1;
          }
    }
    // lane stages (all lanes of an active warp are active)
    if (slot < bpr && r0 + slot < total) {
#pragma unroll
      for (int m = 1; m < 32; m <<= 1) {
        const bool upper = (lane & m) != 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float o = __shfl_xor_sync(0xffffffffu, v[i], m);
          v[i] = upper ? (o - v[i]) : (v[i] + o);
        }
      }
    }
    float* sb = scratch + slot * bsz;
    for (int h = 256; h < bsz; h <<= 1) {
      __syncthreads();
      if (act)
#pragma unroll
        for (int i = 0; i < 8; ++i) sb[e0 + i] = v[i];
      __syncthreads();
      if (act)
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int k = e0 + i;
          const float o = sb[k ^ h];
          v[i] = (k & h) ? (o - v[i]) : (v[i] + o);
        }
    }
    if (act) {
      uint32_t hw[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const __half2 h2 = __floats2half2_rn(v[2 * k] * p.rht_scale, v[2 * k + 1] * p.rht_scale);
        hw[k] = *reinterpret_cast<const uint32_t*>(&h2);
      }
      const int k = blk * bsz + e0;
      uint8_t* dst = xs + beta * p.xs_rs + (k >> 6) * 136 + (k & 63) * 2;
      *reinterpret_cast<uint2*>(dst) = make_uint2(hw[0], hw[1]);
      *reinterpret_cast<uint2*>(dst + 8) = make_uint2(hw[2], hw[3]);
    }
  }
}

// XM: 0 = x' B fragments from global into registers, 1 = x' staged in shared memory,
//     2 = x' computed in shared memory by every CTA from raw x (fused rotation) + in-kernel zeroing
// RP: row tiles per work unit. RP = 2 (batch >= 2, fp32 atomic output): a warp decodes the two
// row tiles of a row pair at the same k tile back to back with the same x' B fragments, halving
// the activation loads per weight.
template <int MODE, int CLO, int CHI, int L, int TB, int REPS, bool DEQ, int XM, int RP>
__global__ void __launch_bounds__(Plan<MODE, CLO, CHI, TB, REPS, (XM != 0)>::NWARP * 32, 1)
    qp_gemv_kernel(const __grid_constant__ GemvParams p) {
  constexpr bool XS = XM != 0;
  using PL = Plan<MODE, CLO, CHI, TB, REPS, XS>;
  constexpr int CMAX = PL::CMAX, NWARP = PL::NWARP;
  static_assert(RP == 1 || (RP == 2 && !DEQ), "row pairs are a GEMV-only (atomic epilogue) variant");
  constexpr int USTAGE = RP * PL::STAGE;          // ring stage: one work unit
  const int NS = p.ns;
  uint8_t* smem = qp_smem;
  uint8_t* tab = smem;
  if (threadIdx.x == 0 && smem_u32(qp_smem) != kDynSmemBase) __trap();
  float* part = reinterpret_cast<float*>(smem + PL::XS_OFF);   // [NWARP][2][256], aliases x' + rings

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#ifdef QP_KERNEL_TIMELINE
  unsigned long long ts[8];   // debug timeline (build with -DQP_KERNEL_TIMELINE, run with QP_TIMELINE=1)
  auto stamp = [&](int k) {
    if (p.timeline) asm volatile("mov.u64 %0, %%clock64;" : "=l"(ts[k]));
  };
  auto flush_stamps = [&](int n) {
    if (p.timeline && lane == 0 && warp < 16)
      for (int k = 0; k < 8; ++k) p.timeline[(blockIdx.x * 16 + warp) * 8 + k] = k < n || k >= 5 ? ts[k] : 0ull;
  };
#else
  auto stamp = [](int) {};
  auto flush_stamps = [](int) {};
#endif
  stamp(0);
  // the compact table words first: their L2 latency then overlaps the rest of the prologue
  TableBuild<REPS, NWARP * 32, PL::ENTRIES> tb;
  tb.load(p.table);
  const int g = lane >> 2, q = lane & 3;
  // tile indices are 32-bit: the host guarantees RT*KT*gridDim < 2^32
  const uint32_t N = (uint32_t)(p.RT / RP) * (uint32_t)p.KT;   // work units (row tile groups x k tiles)
  const uint32_t KT = p.KT;
  // host-computed reciprocals (qp_host.cpp div_magic): no 32-bit integer divisions in the prologue
  auto div_kt = [&](uint32_t x) -> uint32_t { return p.kt_magic ? __umulhi(x, p.kt_magic) : x / KT; };
  auto div_grid = [&](uint32_t x) -> uint32_t { return p.grid_magic ? __umulhi(x, p.grid_magic) : x / gridDim.x; };
  const uint32_t T0 = div_grid(N * blockIdx.x), T1 = div_grid(N * (blockIdx.x + 1));
  const uint32_t nC = T1 - T0;
  const uint32_t a = T0 + nC * warp / NWARP, b = T0 + nC * (warp + 1) / NWARP;
  const int KH = p.KT / 2;
  const long long rowtile_bytes = (long long)KH * 512 * CLO + (long long)(KT - KH) * 512 * CHI;

  // ---- this warp's code ring: NS stages, one tile each, filled by bulk async copies ----
  const uint32_t ring = smem_u32(smem + PL::XS_OFF + p.xs_bytes) + (uint32_t)(warp * NS * USTAGE);
  const uint32_t bars = smem_u32(smem + PL::BAR_OFF) + (uint32_t)(warp * NS * 8);
  uint64_t pol = 0;
  // bytes of k tile kt_ (half-TCQ: c_lo on the first KT/2 k tiles, c_hi on the rest)
  auto tile_bytes = [&](int kt_) -> uint32_t { return 512u * ((CLO == CHI || kt_ < KH) ? CLO : CHI); };
  // issue the copy of the tile at `src` into stage st (lane 0 only)
  auto fetch = [&](const uint8_t* src, uint32_t nbytes, int st, uint32_t dep = 0u) {
    const uint32_t bar = bars + 8u * st;
    mbar_expect_tx(bar, nbytes * RP);
#pragma unroll
    for (int h = 0; h < RP; ++h)   // row tile h of the unit: the next row tile, same k tile
      bulk_g2s(ring + (uint32_t)(st * USTAGE + h * PL::STAGE) + dep, src + h * rowtile_bytes, nbytes, bar, pol);
  };
  uint32_t rt = div_kt(a);                         // row tile group (RP row tiles)
  int kt = (int)(a - rt * KT);
  // the refill cursor: the next tile to be fetched (its address advances by whole tiles: the
  // LAYOUT.md stream is row-tile-major, tiles of a row tile in k order, all contiguous)
  const uint8_t* f_ptr = p.codes + (long long)(RP * rt) * rowtile_bytes +
                         (kt < KH ? (long long)kt * 512 * CLO : (long long)KH * 512 * CLO + (long long)(kt - KH) * 512 * CHI);
  int kt_f = kt;
  auto advance_f = [&]() {
    f_ptr += tile_bytes(kt_f);
    if (++kt_f == (int)KT) {
      kt_f = 0;
      f_ptr += (RP - 1) * rowtile_bytes;             // skip the group's other row tiles
    }
  };
  if (lane == 0) {
#pragma unroll
    for (int st = 0; st < NS; ++st) mbar_init(bars + 8u * st, 1);
    mbar_fence_init();
    pol = l2_evict_first_policy();
    // only the first tile now: the whole grid's first-wave requests then complete before the
    // second wave (issued after the table build) competes with them for HBM
    if (a < b) fetch(f_ptr, tile_bytes(kt_f), 0);
  }
  advance_f();

  // per-row scales of the current row tile, rows g, g+8, g+16, g+24 (prefetched into registers
  // when a row tile starts; consumed when its partial is flushed)
  float sc[4 * RP];
  auto load_scales = [&](uint32_t rt_) {             // rt_: row tile group
    if constexpr (!DEQ) {
#pragma unroll
      for (int i = 0; i < 4 * RP; ++i) sc[i] = __ldg(p.scales + (RP * rt_ + (i >> 2)) * kTileRows + g + 8 * (i & 3));
    }
  };
  if (a < b) load_scales(rt);
  constexpr int NXB = XS ? 4 : 32;                 // B-fragment registers
  uint32_t xb[NXB];
#pragma unroll
  for (int i = 0; i < NXB; ++i) xb[i] = 0u;
  const bool xrow = !DEQ && g < p.batch;           // this lane holds a batch row of x'
  const __half* xlane = p.x + (size_t)g * p.d_in + 64 * q;
  // Everything up to griddepcontrol.wait reads only immutable layer data, so under programmatic
  // dependent launch it overlaps the previous kernel: the code copies are in flight (issued
  // above) while the table words arrive from L2 and are expanded into the replicated image.
  stamp(7);
#ifdef QP_X_EARLY
  // (experiment) wait for the producer and request the first tile's activations before the table
  // expansion, so their L2 latency hides under the 128 KB of shared stores
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (XM == 0 && xrow && a < b) {
    load_x8(xb, xlane + kt * kTileCols);
    load_x8(xb + 8, xlane + kt * kTileCols + 16);
  }
#endif
  tb.store(tab);
  stamp(6);
  for (int st = 1; st < NS; ++st) {                // the rest of the ring's first fill
    if (lane == 0 && a + st < b) fetch(f_ptr, tile_bytes(kt_f), st);
    advance_f();
  }
#ifdef QP_EARLY_TRIGGER
  // (experiment) let the next kernel launch now so its CTAs take SMs as this grid's CTAs exit:
  // same GEMV-alone time, 12% slower C2 step (the next rotation kernel's CTAs then queue behind
  // the GEMV CTAs; profiles/r1/ab_xs_r1.md section 8)
  asm volatile("griddepcontrol.launch_dependents;");
#endif
#ifndef QP_X_EARLY
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
  stamp(5);
  // this lane's x' row in the staged copy (lanes without a batch row read row batch-1: their
  // products land in y columns that are never stored)
  const uint32_t xs_lane = smem_u32(smem + PL::XS_OFF) + (uint32_t)(min(g, p.batch - 1) * p.xs_rs + q * 136);
  if constexpr (XM == 1) {
    // x' (the previous kernel's output) -> padded shared layout, 8 bytes per thread-step
    const int units = p.d_in / 4;                  // 8-byte units per row
    for (int i = tid; i < p.batch * units; i += NWARP * 32) {
      const int row = i / units, k = (i - row * units) * 4;
      const uint2 v = __ldg(reinterpret_cast<const uint2*>(p.x + (size_t)row * p.d_in + k));
      *reinterpret_cast<uint2*>(smem + PL::XS_OFF + row * p.xs_rs + (k >> 6) * 136 + (k & 63) * 2) = v;
    }
  } else if constexpr (XM == 2) {
    if (p.zero_y) {
      // this CTA's share of the fp32 outputs, then arrive on the grid counter; every CTA waits for
      // all arrivals before its first write to y (first_write below)
      const long long gstride = (long long)gridDim.x * NWARP * 32, gme = (long long)blockIdx.x * NWARP * 32 + tid;
      for (int i = 0; i < p.n_out; ++i) {
        const int rows = (p.rt_begin[i + 1] - p.rt_begin[i]) * kTileRows;
        const long long n = (long long)p.batch * rows;
        float* y = reinterpret_cast<float*>(p.y[i]);
        for (long long e = gme; e < n; e += gstride) {
          const int bb = (int)(e / rows);
          y[(size_t)bb * p.ldy[i] + (e - (long long)bb * rows)] = 0.f;
        }
      }
      __syncthreads();
      if (tid == 0) {
        int gen0;
        asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(gen0) : "l"(p.bar_count + 1) : "memory");
        *reinterpret_cast<int*>(smem + PL::BAR_OFF + 1020) = gen0;   // last word of the mbarrier area
        __threadfence();
        if (atomicAdd(p.bar_count, 1) == (int)gridDim.x - 1) {
          p.bar_count[0] = 0;                      // every CTA has arrived: reset, open the barrier
          __threadfence();
          atomicAdd(p.bar_count + 1, 1);
        }
      }
    }
    rotate_x<NWARP>(p, smem + PL::XS_OFF, reinterpret_cast<float*>(smem + PL::XS_OFF + rot_scratch_offset(p.batch, p.xs_rs)));
  } else if (xrow && a < b) {                      // first tile, kappa 0..7
#ifndef QP_X_EARLY
    load_x8(xb, xlane + kt * kTileCols);
    load_x8(xb + 8, xlane + kt * kTileCols + 16);
#endif
  }
  __syncthreads();
  auto scale_of = [&](uint32_t rt_, int row) -> float { return __ldg(p.scales + rt_ * kTileRows + row); };

  stamp(1);
  const uint32_t laneoff = (uint32_t)(lane % REPS) * 4u;
  const uint32_t mulk = (1u << (Dec<MODE, CLO, L, TB, REPS>::KSH > 0 ? Dec<MODE, CLO, L, TB, REPS>::KSH : 0)) + p.zero;
  float acc[2 * RP][4];                            // [row tile of the group][m]
#pragma unroll
  for (int m = 0; m < 2 * RP; ++m)
#pragma unroll
    for (int r = 0; r < 4; ++r) acc[m][r] = 0.f;
  const uint32_t a_rt = rt;

  float hp[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};   // head row-tile partial
  uint32_t cur[4 * CMAX];
  int seg_k0 = kt;                                 // first k tile of the current row-tile segment
  bool y_open = false;                             // XM == 2: the in-kernel zeroing of y is done
  int st = 0;
  uint32_t par = 0;
  for (uint32_t t = a; t < b; ++t) {
    // ---- the unit's stream words: stage st -> registers (c conflict-free 128-bit loads per row
    //      tile), then the row tile's decode + MAC; with RP = 2 the second row tile's words are
    //      read after the first is decoded (same registers) and reuse its x' B fragments ----
    mbar_wait(bars + 8u * st, par);
    int kt_n = kt + 1;
    uint32_t rt_n = rt;
    if (kt_n == (int)KT) { kt_n = 0; ++rt_n; }
    const int c = (CLO == CHI || kt < KH) ? CLO : CHI;
#pragma unroll
    for (int h = 0; h < RP; ++h) {
      const uint32_t src = ring + (uint32_t)(st * USTAGE + h * PL::STAGE) + (uint32_t)lane * 16u;
#pragma unroll
      for (int i = 0; i < CMAX; ++i) {
        if (CLO == CHI || i < c) {
          const uint4 v = lds128(src + i * 512);
          cur[4 * i] = v.x; cur[4 * i + 1] = v.y; cur[4 * i + 2] = v.z; cur[4 * i + 3] = v.w;
        }
      }
      if (h == RP - 1) {
        // The stage is free once every lane's shared loads have returned: a warp reduction over
        // one word of EVERY load of each lane makes lane 0's refill depend on all of them (p.zero
        // == 0 keeps the value unchanged). (ptxas reorders the independent LDS.128s, so the last
        // load in program order need not be the last one issued.)
        uint32_t any = 0;
#pragma unroll
        for (int i = 0; i < CMAX; ++i)
          if (CLO == CHI || i < c) any |= cur[4 * i + 3];
        const uint32_t dep = __reduce_or_sync(0xffffffffu, any & p.zero);
        if (lane == 0 && t + NS < b) fetch(f_ptr, tile_bytes(kt_f), st, dep);
#ifdef QP_L2_PREFETCH
        // warm L2 with the unit after the one just requested (its bulk copy then hits L2)
        if (lane == 0 && t + NS + 1 < b) {
          const uint8_t* nx = f_ptr + tile_bytes(kt_f) + (kt_f + 1 == (int)KT ? (RP - 1) * rowtile_bytes : 0);
#pragma unroll
          for (int hh = 0; hh < RP; ++hh)
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" :: "l"(nx + hh * rowtile_bytes),
                         "r"(tile_bytes(kt_f + 1 == (int)KT ? 0 : kt_f + 1)) : "memory");
        }
#endif
        advance_f();
      }
      const __half* x_hi = (!XS && xrow && h == 0) ? xlane + kt * kTileCols + 32 : nullptr;
      const __half* x_next = (!XS && xrow && h == RP - 1 && t + 1 < b) ? xlane + kt_n * kTileCols : nullptr;
      uint32_t* wout_lane = nullptr;
      int ldw = 0;
      if constexpr (DEQ) {
        ldw = p.d_in / 2;
        wout_lane = reinterpret_cast<uint32_t*>(p.w_out) + (size_t)(rt * kTileRows + g) * ldw + (kt * kTileCols + 64 * q) / 2;
      }
      const uint32_t xs_addr = xs_lane + (uint32_t)(kt * 4 * 136);
      float (&acc_h)[2][4] = *reinterpret_cast<float(*)[2][4]>(&acc[2 * h][0]);
      if (CLO == CHI || kt < KH)
        tile_body<MODE, CLO, L, TB, REPS, DEQ, XS>(cur, laneoff, mulk, xb, acc_h, wout_lane, ldw, x_hi, x_next, xs_addr);
      else
        tile_body<MODE, CHI, L, TB, REPS, DEQ, XS>(cur, laneoff, mulk, xb, acc_h, wout_lane, ldw, x_hi, x_next, xs_addr);
    }
    if (++st == NS) { st = 0; par ^= 1u; }

    if constexpr (!DEQ) {
      if (kt == (int)KT - 1 || t == b - 1) {
        if constexpr (XM == 2) {
          // the grid's in-kernel zeroing of y must be complete before this warp's first write
          if (p.zero_y && !y_open) {
            if (lane == 0) {
              const int gen0 = *reinterpret_cast<const int*>(smem + PL::BAR_OFF + 1020);
              int gen;
              for (;;) {
                asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(gen) : "l"(p.bar_count + 1) : "memory");
                if (gen != gen0) break;
                __nanosleep(32);
              }
            }
            __syncwarp();
            y_open = true;
          }
        }
        const uint32_t rs = rt * KT;                     // (in work units)
        const bool own = (a <= rs) && (b >= rs + KT);
#pragma unroll
        for (int h = 0; h < RP; ++h) {
          const int rth = RP * (int)rt + h;             // row tile
          if (own) {
#pragma unroll
            for (int m = 0; m < 2; ++m)
#pragma unroll
              for (int r = 0; r < 4; ++r) {
                const int row = 16 * m + g + 8 * (r >> 1), bb = 2 * q + (r & 1);
                if (bb < p.batch) store_out(p, rth, row, bb, acc[2 * h + m][r], sc[4 * h + 2 * m + (r >> 1)]);
              }
          } else if (RP == 2 || p.y_atomic) {
            // y was zeroed by the preceding kernel: add this warp's scaled partial straight into it
            // (fire-and-forget RED.ADD.F32; no shared-memory reduction, no barrier). RP = 2 is only
            // launched for the atomic epilogue. fp16 y (y_ws): into the fp32 workspace instead.
            int i = 0;
#pragma unroll 1
            while (i + 1 < p.n_out && rth >= p.rt_begin[i + 1]) ++i;
            float* yb = (p.y_ws ? p.yws[i] : reinterpret_cast<float*>(p.y[i])) + (rth - p.rt_begin[i]) * kTileRows;
#pragma unroll
            for (int m = 0; m < 2; ++m)
#pragma unroll
              for (int r = 0; r < 4; ++r) {
                const int row = 16 * m + g + 8 * (r >> 1), bb = 2 * q + (r & 1);
                if (bb < p.batch)
                  red_add_f32(yb + (size_t)bb * p.ldy[i] + row, acc[2 * h + m][r] * sc[4 * h + 2 * m + (r >> 1)]);
              }
            if (RP == 1 && p.y_ws) {
              // count the k tiles this warp contributed; the warp that completes the row tile's KT
              // converts its 32 rows to fp16 (no waiting anywhere)
              const int nk = kt - seg_k0 + 1;
              __threadfence();
              __syncwarp();
              int last = 0;
              if (lane == 0) last = atomicAdd(p.counters + rth, nk) + nk == (int)KT;
              last = __shfl_sync(0xffffffffu, last, 0);
              if (last) {
                __threadfence();
                __half* yh = reinterpret_cast<__half*>(p.y[i]) + (rth - p.rt_begin[i]) * kTileRows;
                for (int e = lane; e < kTileRows * p.batch; e += 32) {
                  const int bb = e / kTileRows, row = e - bb * kTileRows;
                  yh[(size_t)bb * p.ldy[i] + row] = __float2half_rn(__ldcg(yb + (size_t)bb * p.ldy[i] + row));
                }
                if (lane == 0) p.counters[rth] = 0;      // self-reset for the next launch
              }
            }
          } else if (t + 1 < b) {
            // partial of a row tile shared with other warps / CTAs, kept in registers until every
            // warp has left the main loop (the partial slots alias x' and the code rings). Only the
            // head row tile can end before the range does (middle row tiles are owned); the tail
            // partial simply stays in acc.
#pragma unroll
            for (int m = 0; m < 2; ++m)
#pragma unroll
              for (int r = 0; r < 4; ++r) hp[m][r] = acc[m][r];
          }
        }
        if (own || RP == 2 || p.y_atomic || t + 1 < b) {
#pragma unroll
          for (int m = 0; m < 2 * RP; ++m)
#pragma unroll
            for (int r = 0; r < 4; ++r) acc[m][r] = 0.f;
        }
        if (t + 1 < b) load_scales(rt_n);
        seg_k0 = 0;                                 // the next segment starts at k tile 0
      }
    }
    kt = kt_n; rt = rt_n;
  }
  stamp(2);
#ifndef QP_EARLY_TRIGGER
  // dependents (the next layer's rotation + GEMV) launch once every CTA is past its main loop
  asm volatile("griddepcontrol.launch_dependents;");
#endif
  if (DEQ || nC <= 0 || p.y_atomic) {
    if constexpr (!DEQ) {
      if (nC <= 0) peer_signal(p);                // (the fused all-gather runs the in-order path)
    }
    flush_stamps(3);
    return;
  }

  // ---- reduction of the warp partials: one warp per row tile, no CTA-wide barrier in the loop ----
  __syncthreads();                                    // every warp is done with its code ring
  const bool single_rt = a >= b || div_kt(b - 1) == a_rt;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    float* slot = part + (warp * 2 + h) * 256;
#pragma unroll
    for (int m = 0; m < 2; ++m)
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int row = 16 * m + g + 8 * (r >> 1), bb = 2 * q + (r & 1);
        // one row tile only: its partial is in acc (slot 0); else head in hp, tail in acc
        slot[row * 8 + bb] = h == 0 ? (single_rt ? acc[m][r] : hp[m][r]) : (single_rt ? 0.f : acc[m][r]);
      }
  }
  __syncthreads();
  stamp(4);
  // lane w < NWARP holds warp w's tile range (no divisions inside the loops below)
  const uint32_t my_aw = T0 + nC * (uint32_t)lane / NWARP, my_bw = T0 + nC * (uint32_t)(lane + 1) / NWARP;
  const uint32_t my_frt = my_aw / KT;
  const uint32_t rt_lo = T0 / KT, rt_hi = (T1 - 1) / KT;
  for (uint32_t rt = rt_lo + warp; rt <= rt_hi; rt += NWARP) {
    const uint32_t rs = rt * KT, re = rs + KT;
    // warps touching [rs, re): aw < re && bw > rs, non-empty
    const bool touch = lane < NWARP && my_aw < my_bw && my_aw < re && my_bw > rs;
    const bool sole_owner = touch && my_aw <= rs && my_bw >= re;
    if (__any_sync(0xffffffffu, sole_owner)) continue;   // written directly in the main loop
    const unsigned tmask = __ballot_sync(0xffffffffu, touch);
    const unsigned hmask = __ballot_sync(0xffffffffu, touch && my_frt == rt);   // rt is that warp's first
    // lane handles elements e = lane + 32 k (row = e >> 3, batch = e & 7 = lane & 7)
    const bool act = (lane & 7) < p.batch;
    float v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = 0.f;
#pragma unroll
    for (int w = 0; w < NWARP; ++w) {
      if (tmask & (1u << w)) {
        const float* sl = part + (w * 2 + ((hmask >> w) & 1u ? 0 : 1)) * 256;
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] += sl[lane + 32 * k];
      }
    }
    if (T0 <= rs && T1 >= re) {                          // the whole row tile is in this CTA
      if (act)
#pragma unroll
        for (int k = 0; k < 8; ++k) store_out(p, (int)rt, (lane + 32 * k) >> 3, lane & 7, v[k], scale_of(rt, (lane + 32 * k) >> 3));
      continue;
    }
    // ---- cross-CTA, fast path: y was zeroed by the preceding kernel; every CTA adds its scaled
    //      partial (no waiting; bitwise deterministic when two CTAs share the row tile).
    if (p.y_atomic) {
      if (act) {
        int i = 0;
#pragma unroll 1
        while (i + 1 < p.n_out && (int)rt >= p.rt_begin[i + 1]) ++i;
        float* yb = reinterpret_cast<float*>(p.y[i]) + (size_t)(lane & 7) * p.ldy[i] + (rt - p.rt_begin[i]) * kTileRows;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int row = (lane + 32 * k) >> 3;
          red_add_f32(yb + row, v[k] * scale_of(rt, row));
        }
      }
      continue;
    }
    // ---- cross-CTA, deterministic path: the CTA holding the row tile's first k-tiles (it
    //      finishes them last) sums the others' partials in CTA order; the others publish theirs
    //      and leave without waiting.
    if (rs < T0) {
      // contributor: this row tile is our head (its partial was done first thing)
      if (act)
#pragma unroll
        for (int k = 0; k < 8; ++k) p.ws[(size_t)blockIdx.x * 256 + lane + 32 * k] = v[k];
      __syncwarp();
      if (lane == 0) asm volatile("red.release.gpu.global.add.s32 [%0], 1;" :: "l"(p.counters + rt) : "memory");
      continue;
    }
    const uint32_t c1 = owner_of(re - 1, 0, N, gridDim.x);
    const int need = (int)(c1 - blockIdx.x);
    if (lane == 0) {
      int seen;
      for (;;) {
        asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(seen) : "l"(p.counters + rt) : "memory");
        if (seen >= need) break;
        __nanosleep(64);
      }
      p.counters[rt] = 0;                                 // every contributor has arrived: reset
    }
    __syncwarp();
    if (act) {
      constexpr int kMaxContrib = 8;
      float pv[kMaxContrib][8];
#pragma unroll
      for (int i = 0; i < kMaxContrib; ++i)
        if (i < need)
#pragma unroll
          for (int k = 0; k < 8; ++k) pv[i][k] = __ldcg(p.ws + (size_t)(blockIdx.x + 1 + i) * 256 + lane + 32 * k);
#pragma unroll
      for (int i = 0; i < kMaxContrib; ++i)
        if (i < need)
#pragma unroll
          for (int k = 0; k < 8; ++k) v[k] += pv[i][k];
      for (int i = kMaxContrib; i < need; ++i)
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] += __ldcg(p.ws + (size_t)(blockIdx.x + 1 + i) * 256 + lane + 32 * k);
#pragma unroll
      for (int k = 0; k < 8; ++k) store_out(p, (int)rt, (lane + 32 * k) >> 3, lane & 7, v[k], scale_of(rt, (lane + 32 * k) >> 3));
    }
  }
  __syncthreads();
  stamp(3);
  peer_signal(p);
  flush_stamps(8);
}

template <int MODE, int CLO, int CHI, int L, int TB, int REPS, bool DEQ, int XM, int RP = 1>
cudaError_t launch_one(const GemvParams& prm, int grid, bool pdl, cudaStream_t s) {
  using PL = Plan<MODE, CLO, CHI, TB, REPS, (XM != 0)>;
  const int smem = PL::XS_OFF + (std::max)(prm.xs_bytes + PL::NWARP * prm.ns * RP * PL::STAGE, PL::PART);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(PL::NWARP * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  auto k = qp_gemv_kernel<MODE, CLO, CHI, L, TB, REPS, DEQ, XM, RP>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, PL::SMEM_MAX);
  if (e == cudaSuccess) e = cudaLaunchKernelEx(&cfg, k, prm);
  return e;
}

// Runtime part of the shared-memory plan: stage x' in shared memory when it fits beside at least
// one ring stage per warp (opt-in: QP_XS=1), then as many ring stages (<= 4) as fit. Batch 8
// with the atomic fp32 epilogue and a small decode table uses row-pair units (RP = 2) when d_out
// has an even number of row tiles (QP_RP2_MIN_BATCH overrides the batch threshold; 9 disables).
int env_no_xs();
// the mbarrier area is 1024 B with its last word holding the in-order epilogue's generation: at most
// 127 barriers (8 B each) over all warps, so QP_NS_MAX can never push barriers into the code ring
constexpr int kBarStagesMax = 1016 / 8;
int ns_cap();   // most code-ring stages per warp (QP_NS_MAX; the rest of shared memory is L1)
int rp2_min_batch();
int fused_rht_max_rounds();   // fused rotation: most rounds of in-CTA transforms worth doing
template <int MODE, int CLO, int CHI, int L, int TB, int REPS, bool DEQ>
cudaError_t launch_plan(const GemvParams& prm0, int grid, bool pdl, cudaStream_t s) {
  using PL = Plan<MODE, CLO, CHI, TB, REPS, false>;
  using PX = Plan<MODE, CLO, CHI, TB, REPS, true>;
  GemvParams prm = prm0;
  const int rs = xs_row_stride(prm.d_in);
  const int xs_bytes = rot_scratch_offset(prm.batch, rs);
  if (!DEQ && prm.x_raw) {
    // fused rotation: x' and the rotation scratch beside >= 1 ring stage per warp, and at most
    // fused_rht_max_rounds() rounds of NWARP / (b/256) blocks (else the caller launches the
    // rotation kernel)
    const int spb = prm.rht_block / 256;
    const int scratch = prm.rht_block > 256 ? PX::NWARP * 256 * 4 : 0;
    const int rounds = spb >= 1 && spb <= PX::NWARP ? (prm.batch * (prm.d_in / prm.rht_block) + PX::NWARP / spb - 1) /
                                                          (PX::NWARP / spb) : 1 << 20;
    if (rounds > fused_rht_max_rounds() || xs_bytes + scratch + PX::NWARP * PX::STAGE > PX::AVAIL)
      return cudaErrorNotSupported;
    prm.xs_bytes = xs_bytes + scratch;
    prm.xs_rs = rs;
    prm.ns = (std::min)(4, (PX::AVAIL - prm.xs_bytes) / (PX::NWARP * PX::STAGE));
    return launch_one<MODE, CLO, CHI, L, TB, REPS, false, 2>(prm, grid, pdl, s);
  }
  if (!DEQ && !env_no_xs() && xs_bytes + PX::NWARP * PX::STAGE <= PX::AVAIL) {
    prm.xs_bytes = xs_bytes;
    prm.xs_rs = rs;
    prm.ns = (std::min)(4, (PX::AVAIL - xs_bytes) / (PX::NWARP * PX::STAGE));
    return launch_one<MODE, CLO, CHI, L, TB, REPS, false, 1>(prm, grid, pdl, s);
  }
  prm.xs_bytes = 0;
  prm.xs_rs = 0;
  // row pairs only where they measured faster: batch >= rp2_min_batch() (8) with a small decode
  // table (VQ / NUQ / UNIF), whose ring keeps >= 2 stages of two tiles
  if (!DEQ && prm.y_atomic && !prm.y_ws && prm.batch >= rp2_min_batch() && prm.RT % 2 == 0 && PL::TAB <= 32768 &&
      PL::AVAIL >= PL::NWARP * 2 * 2 * PL::STAGE) {
    prm.ns = (std::min)((std::min)(ns_cap(), kBarStagesMax / PL::NWARP), PL::AVAIL / (PL::NWARP * 2 * PL::STAGE));
    const int units = (prm.RT / 2) * prm.KT;
    if (grid > units) {
      grid = units;
      prm.grid_magic = 0;                          // host reciprocal was for the larger grid
    }
    return launch_one<MODE, CLO, CHI, L, TB, REPS, false, 0, 2>(prm, grid, pdl, s);
  }
  prm.ns = (std::min)((std::min)(ns_cap(), kBarStagesMax / PL::NWARP), PL::AVAIL / (PL::NWARP * PL::STAGE));
  return launch_one<MODE, CLO, CHI, L, TB, REPS, DEQ, 0>(prm, grid, pdl, s);
}

template <int MODE, int CLO, int CHI, int L, int TB, int REPS, bool UNUSED = false>
struct GemvVariant {
  static cudaError_t launch(const GemvParams& prm, int grid, int /*nwarps*/, bool dequant, bool pdl, cudaStream_t s) {
    if (dequant) return launch_plan<MODE, CLO, CHI, L, TB, REPS, true>(prm, grid, pdl, s);
    return launch_plan<MODE, CLO, CHI, L, TB, REPS, false>(prm, grid, pdl, s);
  }
  static void reg() { register_gemv(KernelKey{MODE, CLO, CHI, L, TB, REPS}, &launch); }
};

}  // namespace qp
