// Persistent multi-layer decode engine (qp_multi_fwd): ONE launch runs the whole path -- the
// activation rotations and the fused dequant-GEMVs -- of a list of
// independent layers that share a decode table (e.g. the C2 step: TCQ 2.5 / half-TCQ 3.25 /
// TCQ 4.0 over three Llama shapes, all on the tb = 9 hybrid LUT).
//
// Why (profiles/r2/): a single-layer launch pays a fixed ~2.6 us on B200
// (launch ramp, replicated-table expansion, first tile at full DRAM latency, drain tail) plus a
// dependent rotation kernel. Here
//  * the replicated table is built once per CTA for all layers;
//  * the work units (32 x 256 tiles) of ALL layers form one flat stream-K range split across the
//    persistent CTAs (host-computed CTA ranges, skewed so the CTAs that also run rotation jobs get
//    fewer tiles) and evenly across each CTA's warps -- no per-layer tail;
//  * each warp's code ring simply continues into the next layer's tiles, so the next layer's
//    codes are in flight while the current one drains;
//  * rotation jobs (one (layer, batch row, Hadamard block) each) run on the first CTAs before their
//    tiles; a job writes its slice of x' to global and the last job of a layer bumps that layer's
//    ready flag (monotonic: one increment per launch); a warp waits for the flag once, when it
//    enters the layer -- a device-side flag instead of a kernel boundary;
//  * split row tiles accumulate into a per-layer fp32 workspace with a per-row-tile k-tile counter;
//    the warp completing a row tile writes y (fp32 / fp16, optionally += y) and re-zeroes the
//    workspace and the counter, so no zeroing kernel precedes the launch (self-cleaning).
#pragma once
#include "qp_gemv.cuh"

namespace qp {

// gpu-scope acq_rel / release atomics: with a preceding bar.sync / bar.warp.sync they publish the
// whole CTA's / warp's earlier writes (cumulativity) without a MEMBAR.SC per thread, whose store
// acknowledgements take microseconds while the grid's code copies saturate HBM
__device__ __forceinline__ unsigned atom_add_acqrel(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void red_add_release(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed(unsigned* p, unsigned v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}

// one elected lane of the (converged) warp: the compiler keeps the guarded operands in uniform
// registers (a plain lane == 0 test makes it move them through a per-lane waterfall loop)
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}" : "=r"(pred));
  return pred != 0;
}

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <int MODE, int L, int TB, int REPS, int CMIN, int CMAX>
struct EPlan {
  static constexpr int ENTRIES = MODE == DEC_TCQ_PRESIGNED ? (2 << TB) : MODE == DEC_LUT2 ? (1 << CMAX) : (1 << TB);
  static constexpr int TAB = ENTRIES * REPS * 4 < 4096 ? 4096 : ENTRIES * REPS * 4;
  static constexpr int SMEM_MAX = 232448;
  static constexpr int STAGE = 512 * CMAX;
#ifndef QP_ENG_WARPS
#define QP_ENG_WARPS 16
#endif
  static constexpr int NWARP = CMAX <= 8 ? QP_ENG_WARPS : (QP_ENG_WARPS < 12 ? QP_ENG_WARPS : 12);
  static constexpr int BAR_OFF = TAB;                 // <= 16 warps x 4 stages x 8 B
  static constexpr int RING_OFF = TAB + 1024;
  static constexpr int AVAIL = SMEM_MAX - RING_OFF;
  static_assert(AVAIL >= NWARP * STAGE, "engine shared-memory plan does not fit");
  // ring stages per warp, a compile-time constant (the ring index arithmetic of every tile folds):
  // 2 where they fit (the rest of shared memory is L1 for the activations), else 1
  static constexpr int NS = AVAIL / (NWARP * STAGE) >= 2 ? 2 : 1;
  static_assert(MODE != DEC_LUT2 || CMIN == CMAX, "LUT2 tables depend on c: one width per engine variant");
};

// One rotation job: x'[beta][blk*b .. (blk+1)*b) = (1/sqrt(b)) H_b (D x)[...] for one layer, by the
// whole CTA, through `scr` (b fp32, shared memory that is not live yet). The operations are those
// of qp_rht_kernel<8> in the same order (3 butterfly stages in registers, 5 by shfl.xor, the rest
// through shared memory; fp32; one RNE rounding), so x' is bitwise the rotation kernel's.
template <int NWARP>
__device__ __forceinline__ void engine_rotate(const EngOp& o, int x_dtype, int beta, int blk, float* scr) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int bsz = o.rht_block, nseg = bsz >> 8;
  for (int seg = warp; seg < nseg; seg += NWARP) {
    const int e0 = seg * 256 + lane * 8;                       // element within the block
    const size_t base = (size_t)beta * o.d_in + (size_t)blk * bsz + e0;
    float v[8];
    if (x_dtype == 0) {
      const uint4 u = *reinterpret_cast<const uint4*>(reinterpret_cast<const __half*>(o.x_raw) + base);
      const __half2* h = reinterpret_cast<const __half2*>(&u);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float2 f = __half22float2(h[k]);
        v[2 * k] = f.x;
        v[2 * k + 1] = f.y;
      }
    } else if (x_dtype == 1) {
      const __nv_bfloat16* xb = reinterpret_cast<const __nv_bfloat16*>(o.x_raw) + base;
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = __bfloat162float(xb[i]);
    } else {
      const float4 f0 = *reinterpret_cast<const float4*>(reinterpret_cast<const float*>(o.x_raw) + base);
      const float4 f1 = *(reinterpret_cast<const float4*>(reinterpret_cast<const float*>(o.x_raw) + base) + 1);
      v[0] = f0.x; v[1] = f0.y; v[2] = f0.z; v[3] = f0.w; v[4] = f1.x; v[5] = f1.y; v[6] = f1.z; v[7] = f1.w;
    }
    const int gi = blk * bsz + e0;                               // 8 | gi: one sign word
    const uint32_t sw = __ldg(o.rht_signs + (gi >> 5)) >> (gi & 31);
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
#pragma unroll
    for (int m = 1; m < 32; m <<= 1) {
      const bool upper = (lane & m) != 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float ov = __shfl_xor_sync(0xffffffffu, v[i], m);
        v[i] = upper ? (ov - v[i]) : (v[i] + ov);
      }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) scr[e0 + i] = v[i];
  }
  // strides 256 .. b/2 in place: (lower, upper) -> (lower + upper, lower - upper)
  const int NT = NWARP * 32;
  for (int h = 256; h < bsz; h <<= 1) {
    __syncthreads();
    for (int i = tid; i < bsz / 2; i += NT) {
      const int lo = ((i & ~(h - 1)) << 1) | (i & (h - 1)), hi = lo | h;
      const float a0 = scr[lo], a1 = scr[hi];
      scr[lo] = a0 + a1;
      scr[hi] = a0 - a1;
    }
  }
  __syncthreads();
  __half* out = o.xr + (size_t)beta * o.d_in + (size_t)blk * bsz;
  for (int i = tid; i < bsz / 8; i += NT) {
    uint4 u;
    __half2* h2 = reinterpret_cast<__half2*>(&u);
#pragma unroll
    for (int k = 0; k < 4; ++k) h2[k] = __floats2half2_rn(scr[8 * i + 2 * k] * o.rht_scale, scr[8 * i + 2 * k + 1] * o.rht_scale);
    *reinterpret_cast<uint4*>(out + 8 * i) = u;
  }
}

// runtime c -> f(std::integral_constant<int, C>) for C in [CMIN, CMAX] (every register array of the
// tile then has compile-time extent and indices)
template <int CMIN, int CMAX, class F>
__device__ __forceinline__ void c_dispatch(int c, F&& f) {
  if constexpr (CMIN == CMAX) {
    f(std::integral_constant<int, CMIN>{});
  } else {
    if (c == CMIN) f(std::integral_constant<int, CMIN>{});
    else c_dispatch<CMIN + 1, CMAX>(c, f);
  }
}

#ifdef QP_ENG_TIMELINE
// experiment builds only (-DQP_ENG_TIMELINE): globaltimer stamps of warp 0 of every CTA
__device__ unsigned long long g_eng_tl[kMaxEngCtas][8];
__device__ unsigned long long g_eng_wl[kMaxEngCtas][16];   // per-warp main-loop end
#define QP_TL(k) do { if (threadIdx.x == 0) { unsigned long long t_; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_)); g_eng_tl[blockIdx.x][k] = t_; } } while (0)
#else
#define QP_TL(k) do { } while (0)
#endif

// Fused all-gather store (qp_multi_fwd_sharded_p2p): the final value of (batch row bb, row) of layer o
// into every rank's y_full. (Inline on purpose: as __noinline__ calls these helpers made every engine
// variant 1-6 % slower -- call-site register constraints; profiles/r2/v5/peer_helpers_ab.txt.)
__device__ __forceinline__ void store_peers(const EngParams& p, const EngOp& o, int bb, int row, float v) {
  const size_t eb = p.y_f32 ? 4 : 2;
  const size_t off = (size_t)(reinterpret_cast<const char*>(o.y) - p.peer_base[p.peer_rank]) +
                     (((size_t)bb * p.n_peers + p.peer_rank) * o.d_out + row) * eb;
#pragma unroll 1
  for (int k = 0; k < p.n_peers; ++k) {
    if (p.y_f32) *reinterpret_cast<float*>(p.peer_base[k] + off) = v;
    else *reinterpret_cast<__half*>(p.peer_base[k] + off) = __float2half_rn(v);
  }
}

// The fused all-gather's launch-exit protocol: arrive = this CTA's peer stores fenced before its arrival
// on the exit counter; deliver = the last CTA bumps this rank's delivery counter on every rank.
// Flag array of a rank (unsigned[2 * world + 1], as qp_linear_fwd_sharded_p2p's): [k] deliveries from
// rank k, [world] rounds this rank has consumed, [world + 1 + k] rounds rank k has entered. One engine
// launch = one round: its CTA 0 announces the entry on every rank once the launch may run (after
// griddepcontrol.wait: this rank's earlier stream work, incl. readers of the previous round's y_full,
// is done); a warp's first peer store waits until every rank has entered the round; the last CTA out
// delivers to every rank, waits for every rank's delivery and counts the round consumed -- so the
// kernel's completion means every y_full holds every rank's rows (no enter / wait kernels: the PDL
// chain between consecutive engine launches stays intact). A peer that never shows traps after 20 s.
constexpr unsigned long long kEngPeerTimeoutNs = 20ull * 1000 * 1000 * 1000;
__device__ __forceinline__ unsigned long long eng_gtimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned ld_acquire_sys_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// every rank's flag [base + k] >= want (k = 0 .. world-1)
__device__ __forceinline__ void peer_wait_all(const unsigned* local, int base, int world, unsigned want) {
  const unsigned long long t0 = eng_gtimer_ns();
#pragma unroll 1
  for (int k = 0; k < world; ++k)
    while ((int)(ld_acquire_sys_u32(local + base + k) - want) < 0) {
      if (eng_gtimer_ns() - t0 > kEngPeerTimeoutNs) __trap();
      __nanosleep(64);
    }
}
__device__ __forceinline__ void peer_enter(const EngParams& p) {
  const int world = p.n_peers;
#pragma unroll 1
  for (int k = 0; k < world; ++k) atomicAdd_system(p.peer_flag[k] + world + 1 + p.peer_rank, 1u);
}
__device__ __forceinline__ void peer_fence() { __threadfence_system(); }
__device__ __forceinline__ void peer_deliver(const EngParams& p) {
  __threadfence_system();
#pragma unroll 1
  for (int k = 0; k < p.n_peers; ++k) atomicAdd_system(p.peer_flag[k] + p.peer_rank, 1u);
  // every rank's rows of this round have arrived here, then the round is consumed
  unsigned* local = p.peer_flag[p.peer_rank];
  const unsigned round = local[p.n_peers] + 1u;
  peer_wait_all(local, 0, p.n_peers, round);
  local[p.n_peers] = round;
  __threadfence_system();
}

// RP: row tiles per work unit. RP = 2 (batch >= 4): a unit is the two row tiles of a row pair at one
// k tile, decoded back to back with the same activation fragments -- half the x' loads, which are
// the batch-8 bottleneck (MIO: 4 KB of x' per 32x256 tile at batch 8).
template <int MODE, int L, int TB, int REPS, int CMIN, int CMAX, int RP>
__global__ void __launch_bounds__(EPlan<MODE, L, TB, REPS, CMIN, CMAX>::NWARP * 32, 1)
    qp_engine_kernel(const __grid_constant__ EngParams p) {
  using PL = EPlan<MODE, L, TB, REPS, CMIN, CMAX>;
  constexpr int NWARP = PL::NWARP;
  constexpr int NS = PL::NS;
  uint8_t* smem = qp_smem;
  if (threadIdx.x == 0 && smem_u32(qp_smem) != kDynSmemBase) __trap();
  // warp index through a lane-0 broadcast: provably warp-uniform to the compiler, so the ring /
  // range / fetch arithmetic derived from it lives in uniform registers (no per-copy waterfall loop
  // to feed the bulk copy's uniform operands)
  const int tid = threadIdx.x, lane = tid & 31, warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  const int g = lane >> 2, q = lane & 3;
  QP_TL(0);

  TableBuild<REPS, NWARP * 32, PL::ENTRIES> tbl;
  tbl.load(p.table);

  // ---- this warp's units: [a, b) of the flat order (host-computed CTA ranges, split evenly over
  //      the CTA's warps). A unit is RP row tiles (a row pair for RP = 2) at one k tile ----------
  const uint32_t T0 = p.cta_begin[blockIdx.x], T1 = p.cta_begin[blockIdx.x + 1];
  const uint32_t nC = T1 - T0;
  const uint32_t a = T0 + nC * warp / NWARP, b = T0 + nC * (warp + 1) / NWARP;
  // packed geometry of a layer: KT | KH << 8 | c_lo << 16 | c_hi << 24 (KT <= 255, c <= 10)
  auto pack = [&](int o_) -> uint32_t {
    const EngOp& o = p.op[o_];
    return (uint32_t)o.KT | ((uint32_t)o.KH << 8) | ((uint32_t)o.c_lo << 16) | ((uint32_t)o.c_hi << 24);
  };
  auto units_of = [&](int o_) -> uint32_t { return (uint32_t)(p.op[o_].RT / RP) * (uint32_t)p.op[o_].KT; };
  // decode cursor of unit a: layer oi, row group rt (row tiles RP*rt ..), k tile kt, geometry opk,
  // units left in the layer
  int oi = 0;
  while (oi + 1 < p.n_ops && a >= p.op[oi + 1].tile0) ++oi;
  uint32_t rt, kt, opk = 0, left = 0;
  {
    const uint32_t loc = a - p.op[oi].tile0, KT_ = (uint32_t)p.op[oi].KT;
    rt = loc / KT_;
    kt = loc - rt * KT_;
    if (a < b) {
      opk = pack(oi);
      left = units_of(oi) - loc;
    }
  }

  // ---- the code ring (one tile per stage; the tile sequence is unit-major, h = 0..RP-1 inside) --
  // (from the constant dynamic-shared-memory base checked above: rematerialising these from the
  // generic pointer cost an S2R SR_CgaCtaId + LEA in every tile of the loop)
  const uint32_t ring = kDynSmemBase + PL::RING_OFF + (uint32_t)(warp * NS * PL::STAGE);
  const uint32_t bars = kDynSmemBase + PL::BAR_OFF + (uint32_t)(warp * NS * 8);
  // Copy tile h_ of the unit d units after the decode cursor (oi_, rt_, kt_, left_, opk_) into stage
  // st (an elected lane issues). RP = 1: f_ptr is the address following the previous copy (inside a
  // layer a warp's tiles are contiguous, row-tile-major), so the next copy starts there; the first
  // copy, a copy into a later layer and every RP = 2 copy compute the address.
  const uint8_t* f_ptr = nullptr;
  const uint64_t pol = l2_evict_first_policy();   // once: a per-copy createpolicy costs ~6 issue slots a tile
  auto fetch_ahead = [&](int st, uint32_t dep, uint32_t d, uint32_t h_, bool cont, int oi_, uint32_t rt_, uint32_t kt_,
                         uint32_t left_, uint32_t opk_) {
    const uint8_t* src;
    if (RP == 1 && cont && d < left_) {        // same layer as the previous copy: contiguous
      const uint32_t KT_ = opk_ & 0xffu;
      kt_ += d;
      while (kt_ >= KT_) kt_ -= KT_;
      src = f_ptr;
    } else {
      if (d < left_) {
        const uint32_t KT_ = opk_ & 0xffu;
        kt_ += d;
        while (kt_ >= KT_) { kt_ -= KT_; ++rt_; }
      } else {                                 // in a later layer
        d -= left_;
        ++oi_;
        while (oi_ + 1 < p.n_ops && d >= units_of(oi_)) {
          d -= units_of(oi_);
          ++oi_;
        }
        opk_ = pack(oi_);
        rt_ = d / (opk_ & 0xffu);
        kt_ = d - rt_ * (opk_ & 0xffu);
      }
      const EngOp& o = p.op[oi_];
      const uint32_t KH_ = (opk_ >> 8) & 0xffu, clo = (opk_ >> 16) & 0xffu, chi = opk_ >> 24;
      src = o.codes + (long long)(RP * rt_ + h_) * o.rowtile_bytes +
            (kt_ < KH_ ? kt_ * 512u * clo : KH_ * 512u * clo + (kt_ - KH_) * 512u * chi);
    }
    const uint32_t KH_ = (opk_ >> 8) & 0xffu;
    const uint32_t nb = 512u * (kt_ < KH_ ? (opk_ >> 16) & 0xffu : opk_ >> 24);
    if (elect_one()) {
      const uint32_t bar = bars + 8u * st;
      mbar_expect_tx(bar, nb);
      bulk_g2s(ring + (uint32_t)(st * PL::STAGE) + dep, src, nb, bar, pol);
    }
    f_ptr = src + nb;
  };
  // the tile sequence position pos (relative to unit a's first tile) -> (units ahead, h)
  const uint32_t ntiles = (b - a) * RP;

  // ---- ordering with earlier work ----------------------------------------------------------------
  // Default: griddepcontrol.wait (x may come from the preceding kernel; y may be read by it).
  // QP_INDEPENDENT (the caller guarantees that no work still running on the stream touches this
  // call's x or y): no wait on the preceding kernel -- consecutive independent calls overlap -- only
  // on the previous launch of THIS launch group (its workspace, counters and x' scratch): every CTA
  // takes an entry ticket (64-bit, monotonic), ticket / gridDim.x is the launch index, and the CTA
  // waits until that many launches of the group have exited (gen64[1], bumped by the last CTA out).
  unsigned long long* gen64 = reinterpret_cast<unsigned long long*>(p.gen + 2);   // [0] entry, [1] exits
  auto order_before = [&]() {
    // every launch takes its tickets (so launch indices count dependent and independent launches)
    const unsigned long long ticket = tid == 0 ? atomicAdd(gen64, 1ull) : 0ull;
    if (!p.independent) {
      asm volatile("griddepcontrol.wait;" ::: "memory");
      return;
    }
    if (tid == 0) {
      const unsigned long long idx = ticket / gridDim.x;
      for (;;) {
        unsigned long long done;
        asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(done) : "l"(gen64 + 1) : "memory");
        if ((long long)(done - idx) >= 0) break;
        __nanosleep(64);
      }
    }
    __syncthreads();
  };

  // ---- rotation jobs (the first CTAs): x' of every layer, before this CTA's own tiles ------------
  const bool rotor = (int)blockIdx.x < p.total_jobs;
  if (rotor) {
    order_before();
    QP_TL(1);
    for (int j = blockIdx.x; j < p.total_jobs; j += gridDim.x) {
      int jo = 0;
      while (jo + 1 < p.n_ops && j >= p.op[jo + 1].job0) ++jo;
      const EngOp& o = p.op[jo];
      const int jl = j - o.job0, nblk = o.d_in / o.rht_block;
      const int beta = jl / nblk, blk = jl - beta * nblk;
      engine_rotate<NWARP>(o, p.x_dtype, beta, blk, reinterpret_cast<float*>(smem));   // table / ring area: not live
      QP_TL(7);
      __syncthreads();
      if (tid == 0) red_add_release(o.ready, 1u);               // one more of the layer's jobs done
    }
    __syncthreads();                                            // scratch reads done before the table build
  }
  if (lane == 0) {
#pragma unroll 1
    for (int st = 0; st < NS; ++st) mbar_init(bars + 8u * st, 1);
    mbar_fence_init();
    *reinterpret_cast<volatile unsigned*>(smem + PL::BAR_OFF + 512 + 4 * warp) = 0u;   // peer gate
  }
  __syncwarp();
  if (a < b) fetch_ahead(0, 0u, 0u, 0u, false, oi, rt, kt, left, opk);
  QP_TL(2);
  tbl.store(smem);
  if (!p.late_stages)
    for (int st = 1; st < NS && (uint32_t)st < ntiles; ++st)
      fetch_ahead(st, 0u, (uint32_t)st / RP, (uint32_t)st % RP, true, oi, rt, kt, left, opk);
  if (!rotor) order_before();
  if (p.n_peers > 0 && blockIdx.x == 0 && tid == 0) peer_enter(p);   // this rank entered the round
  QP_TL(3);
  __syncthreads();

  const uint32_t laneoff = (uint32_t)(lane % REPS) * 4u;
  const uint32_t mulk = (1u << (Dec<MODE, CMIN, L, TB, REPS>::KSH > 0 ? Dec<MODE, CMIN, L, TB, REPS>::KSH : 0)) + p.zero;
#ifdef QP_ENG_EXP_XROW1
  const bool xrow = g < 1;   // experiment: activation loads of batch row 0 only (wrong results for batch > 1)
#else
  const bool xrow = g < p.batch;
#endif
  // Register economy: the main loop keeps only a packed copy of the current layer's geometry and
  // the tiles left in it; every other per-layer field is read from the parameter bank where it is
  // needed, through an index the compiler cannot hoist (shfl of the layer index), so no per-layer
  // address set stays live across the decode.
  auto opaque = [&](int v) -> int { return __shfl_sync(0xffffffffu, v, 0); };
  // fused all-gather: before this warp's first peer store of the launch, every rank has entered the
  // round (a warp-private shared word remembers it; the upper half of the barrier area is unused)
  volatile unsigned* gate = reinterpret_cast<volatile unsigned*>(smem + PL::BAR_OFF + 512) + warp;
  auto peer_gate = [&]() {
    if (*gate == 0u) {
      const unsigned* local = p.peer_flag[p.peer_rank];
      peer_wait_all(local, p.n_peers + 1, p.n_peers, local[p.n_peers] + 1u);
      *gate = 1u;
    }
  };
  // wait until layer o_'s x' is complete in this launch (`ready` counts its finished rotation jobs
  // and is reset by the last CTA out): acquire polling
  auto enter_op = [&](int o_) {
    const EngOp& o = p.op[o_];
    if (o.njobs > 0) {
      // every poll is an acquire load: the load that sees the count complete is the acquire (one
      // L2 round trip less than relaxed polling + a separate acquire)
      const unsigned want = (unsigned)o.njobs;
#ifdef QP_ENG_RELAXED_POLL
      if (*reinterpret_cast<volatile const unsigned*>(o.ready) < want) {
        for (;;) {
          __nanosleep(32);
          if (*reinterpret_cast<volatile const unsigned*>(o.ready) >= want) break;
        }
      }
      (void)ld_acquire_u32(o.ready);
#else
      while (ld_acquire_u32(o.ready) < want) __nanosleep(32);
#endif
    }
  };
  float sc[RP][4];
  auto load_scales = [&](int o_, uint32_t rt_) {
#pragma unroll
    for (int h = 0; h < RP; ++h) {
      const float* s = p.op[o_].scales + (RP * rt_ + h) * kTileRows + g;
#pragma unroll
      for (int i = 0; i < 4; ++i) sc[h][i] = __ldg(s + 8 * i);
    }
  };
  uint32_t xb[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) xb[i] = 0u;
  // this lane's x' row (g) and column group (q) of layer o_
  auto xlane = [&](int o_) -> const __half* { return p.op[o_].xr + (size_t)g * p.op[o_].d_in + 64 * q; };
  const __half* xl = nullptr;            // this lane's x' row of the current layer
  if (a < b) {
    enter_op(oi);
    QP_TL(4);
    if (p.late_stages)
      for (int st = 1; st < NS && (uint32_t)st < ntiles; ++st)
        fetch_ahead(st, 0u, (uint32_t)st / RP, (uint32_t)st % RP, true, oi, rt, kt, left, opk);
    load_scales(oi, rt);
    xl = xlane(oi);
    if (xrow) {
      load_x8_coh(xb, xl + kt * kTileCols);
      load_x8_coh(xb + 8, xl + kt * kTileCols + 16);
    }
  }
  float acc[RP][2][4];
#pragma unroll
  for (int h = 0; h < RP; ++h)
#pragma unroll
    for (int m = 0; m < 2; ++m)
#pragma unroll
      for (int r = 0; r < 4; ++r) acc[h][m][r] = 0.f;
  int seg_k0 = (int)kt;
  int st = 0;
  uint32_t par = 0;
  // The loop runs over *runs*: consecutive units of one row group at one step width c (a row group
  // is one run, or two for half-TCQ), each run a compile-time-c inner loop whose per-tile work is
  // only the ring wait, the stage's shared loads, the next copy and the decode; row / layer
  // transitions and the epilogue happen between runs.
  for (uint32_t t = a; t < b;) {
    const uint32_t KT = opk & 0xffu, KH = (opk >> 8) & 0xffu;
    const int c = kt < KH ? (int)((opk >> 16) & 0xffu) : (int)(opk >> 24);
    const uint32_t kend = kt < KH ? KH : KT;                 // the run ends at k tile kend (exclusive)
    const uint32_t n = min(kend - kt, b - t);
    const bool run_row_end = kt + n == KT;
    c_dispatch<CMIN, CMAX>(c, [&](auto CC) {
      constexpr int C = decltype(CC)::value;
#pragma unroll 1
      for (uint32_t i = 0; i < n; ++i) {
        const uint32_t tt = t + i;
        const bool row_end = kt + 1 == KT;
        // activations: the second half of this k tile at the unit's first tile; the first half of
        // the next unit's k tile mid-way through its last tile, when that unit is in the same layer
        const __half* x_nx =
            (xrow && tt + 1 < b && left != 1u) ? xl + (row_end ? 0u : kt + 1) * kTileCols : nullptr;
#pragma unroll
        for (int h = 0; h < RP; ++h) {
          mbar_wait(bars + 8u * st, par);
          const uint32_t src = ring + (uint32_t)(st * PL::STAGE) + (uint32_t)lane * 16u;
          uint32_t cur[4 * C];
#pragma unroll
          for (int w = 0; w < C; ++w) {
            const uint4 v = lds128(src + w * 512);
            cur[4 * w] = v.x; cur[4 * w + 1] = v.y; cur[4 * w + 2] = v.z; cur[4 * w + 3] = v.w;
          }
          // the stage is free once every lane's shared loads have returned: the warp reduction
          // depends on one word of EVERY load (ptxas reorders the independent LDS.128s, so the last
          // one in program order is not the last issued: depending on it alone let the refill
          // overwrite words still in flight -- a race the shorter fast-path issue exposed)
          uint32_t any = 0;
#pragma unroll
          for (int w = 0; w < C; ++w) any |= cur[4 * w + 3];
          const uint32_t dep = __reduce_or_sync(0xffffffffu, any & p.zero);
          const uint32_t pos = (tt - a) * RP + h + NS;         // the tile sequence position to fetch
#ifdef QP_ENG_NO_FASTPATH
          if (false) {
#else
          if (RP == 1 && i + (uint32_t)NS < n) {
#endif
            // the tile NS ahead is in this run: same width C, right after the previous copy
            if (elect_one()) {
              const uint32_t bar = bars + 8u * st;
              mbar_expect_tx(bar, 512u * C);
              bulk_g2s(ring + (uint32_t)(st * PL::STAGE) + dep, f_ptr, 512u * C, bar, pol);
            }
            f_ptr += 512u * C;
          } else if (pos < ntiles) {
            fetch_ahead(st, dep, (h + NS) / RP, (h + NS) % RP, true, oi, rt, kt, left, opk);
          }
          const __half* x_hi = (xrow && h == 0) ? xl + kt * kTileCols + 32 : nullptr;
          const __half* x_next = h == RP - 1 ? x_nx : nullptr;
          tile_body<MODE, C, L, TB, REPS, false, false, true>(cur, laneoff, mulk, xb, acc[h], nullptr, 0, x_hi, x_next,
                                                             0u);
          if (++st == NS) { st = 0; par ^= 1u; }
        }
        --left;
        ++kt;
      }
    });
    t += n;
    --kt;                                  // kt = the run's last k tile (the epilogue's view)
    const bool row_end = run_row_end;
    const bool op_end = row_end && left == 0u;
    if (row_end || t == b) {
      // ---- end of this warp's segment of row group rt: each of its RP row tiles ----
      const int oe = opaque(oi);
      const int d_out = p.op[oe].d_out;
#pragma unroll
      for (int h = 0; h < RP; ++h) {
        const uint32_t rth = RP * rt + h;                   // row tile
        if (seg_k0 == 0 && row_end) {                       // the whole row tile: store directly
          void* yv = p.op[oe].y;
#pragma unroll
          for (int m = 0; m < 2; ++m)
#pragma unroll
            for (int r = 0; r < 4; ++r) {
              const int row = 16 * m + g + 8 * (r >> 1), bb = 2 * q + (r & 1);
              if (bb < p.batch) {
                const float v = acc[h][m][r] * sc[h][2 * m + (r >> 1)];
                if (p.n_peers > 0) {
                  peer_gate();
                  store_peers(p, p.op[oe], bb, rth * kTileRows + row, v);
                } else {
                  const size_t e = (size_t)bb * d_out + rth * kTileRows + row;
                  if (p.y_f32) {
                    float* y = reinterpret_cast<float*>(yv) + e;
                    *y = p.y_accum ? *y + v : v;
                  } else {
                    reinterpret_cast<__half*>(yv)[e] = __float2half_rn(v);
                  }
                }
              }
            }
        } else {
          float* wsb = p.op[oe].ws + rth * kTileRows;
#pragma unroll
          for (int m = 0; m < 2; ++m)
#pragma unroll
            for (int r = 0; r < 4; ++r) {
              const int row = 16 * m + g + 8 * (r >> 1), bb = 2 * q + (r & 1);
              if (bb < p.batch) red_add_f32(wsb + (size_t)bb * d_out + row, acc[h][m][r] * sc[h][2 * m + (r >> 1)]);
            }
          const int nk = (int)kt - seg_k0 + 1;
          unsigned* cnt = reinterpret_cast<unsigned*>(p.op[oe].counters + rth);
          __syncwarp();
          int done = 0;
          if (lane == 0) done = atom_add_acqrel(cnt, (unsigned)nk) + (unsigned)nk == KT;
          done = __shfl_sync(0xffffffffu, done, 0);
          if (done) {
            // every k tile of row tile rth is in the workspace: write y, re-zero the workspace
            __syncwarp();
            void* yv = p.op[oe].y;
            for (int e = lane; e < kTileRows * p.batch; e += 32) {
              const int bb = e >> 5, row = e & 31;
              float* wp = wsb + (size_t)bb * d_out + row;
              const float v = __ldcg(wp);
              __stcg(wp, 0.f);
              const size_t ye = (size_t)bb * d_out + rth * kTileRows + row;
              if (p.n_peers > 0) {
                peer_gate();
                store_peers(p, p.op[oe], bb, rth * kTileRows + row, v);
              } else if (p.y_f32) {
                float* y = reinterpret_cast<float*>(yv) + ye;
                *y = p.y_accum ? *y + v : v;
              } else {
                reinterpret_cast<__half*>(yv)[ye] = __float2half_rn(v);
              }
            }
            if (lane == 0) st_relaxed(cnt, 0u);
          }
        }
      }
#pragma unroll
      for (int h = 0; h < RP; ++h)
#pragma unroll
        for (int m = 0; m < 2; ++m)
#pragma unroll
          for (int r = 0; r < 4; ++r) acc[h][m][r] = 0.f;
      seg_k0 = 0;
    }
    // ---- advance to the next run ----
    if (row_end) {
      kt = 0;
      ++rt;
      if (op_end) {
        ++oi;
        rt = 0;
        if (t < b) {
          const int on = opaque(oi);
          opk = pack(on);
          left = units_of(on);
          enter_op(on);
          xl = xlane(on);
          if (xrow) {
            load_x8_coh(xb, xl);
            load_x8_coh(xb + 8, xl + 16);
          }
        }
      }
      if (t < b) load_scales(opaque(oi), rt);
    } else {
      ++kt;
    }
  }
  QP_TL(5);
#ifdef QP_ENG_TIMELINE
  if (lane == 0 && warp < 16) {
    unsigned long long t_;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
    g_eng_wl[blockIdx.x][warp] = t_;
  }
#endif
  asm volatile("griddepcontrol.launch_dependents;");
  // the last CTA out resets the launch's ready counters (every CTA is past its waits)
  __syncthreads();
  if (tid == 0) {
    if (p.n_peers > 0) peer_fence();             // this CTA's peer stores before its arrival
    if (atom_add_acqrel(p.gen, 1u) == gridDim.x - 1) {
      // every CTA's stores are in every y_full: deliver (fence / relaxed atomic / fence chain, as
      // peer_signal; qp_peer_wait_kernel consumes one delivery per engine launch and rank)
      if (p.n_peers > 0) peer_deliver(p);
      for (int o_ = 0; o_ < p.n_ops; ++o_) st_relaxed(p.op[o_].ready, 0u);
      st_relaxed(p.gen, 0u);
      // this launch of the group has exited (QP_INDEPENDENT launches of the group wait for it)
      asm volatile("red.release.gpu.global.add.u64 [%0], 1;" :: "l"(gen64 + 1) : "memory");
    }
  }
  QP_TL(6);
}

template <int MODE, int L, int TB, int REPS, int CMIN, int CMAX>
struct EngineVariant {
  static cudaError_t launch(const EngParams& prm0, int grid, bool pdl, cudaStream_t s) {
    using PL = EPlan<MODE, L, TB, REPS, CMIN, CMAX>;
    EngParams prm = prm0;
    prm.ns = PL::NS;   // (QP_NS_MAX applies to the per-layer kernel only)
    int smem = PL::RING_OFF + PL::NWARP * prm.ns * PL::STAGE;
    smem = (std::max)(smem, prm.rot_scratch_bytes);
    if (smem > PL::SMEM_MAX) return cudaErrorInvalidValue;
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
    // row pairs only for the small-table schemes: the TCQ decode is register-bound, and a second set of
    // accumulators + scales cost more than the halved activation loads save (measured: C2 at batch 4
    // +32%, batch 8 +12%; VQ-3 / NUQ-4 at batch 8 -9%, profiles/r2/ab_rp.md)
    void (*k)(EngParams) = qp_engine_kernel<MODE, L, TB, REPS, CMIN, CMAX, 1>;
    if constexpr (MODE == DEC_LUT2) {
      if (prm.rp == 2) k = qp_engine_kernel<MODE, L, TB, REPS, CMIN, CMAX, 2>;
    } else {
      prm.rp = 1;
    }
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, PL::SMEM_MAX);
    if (e == cudaSuccess) e = cudaLaunchKernelEx(&cfg, k, prm);
    return e;
  }
  static void reg() { register_engine(EngineKey{MODE, L, TB, REPS, CMIN, CMAX}, &launch); }
};

}  // namespace qp
