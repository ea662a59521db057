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
  static constexpr int NWARP = CMAX <= 8 ? 16 : 12;
  static constexpr int BAR_OFF = TAB;                 // <= 16 warps x 4 stages x 8 B
  static constexpr int RING_OFF = TAB + 1024;
  static constexpr int AVAIL = SMEM_MAX - RING_OFF;
  static_assert(AVAIL >= NWARP * STAGE, "engine shared-memory plan does not fit");
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

template <int MODE, int L, int TB, int REPS, int CMIN, int CMAX>
__global__ void __launch_bounds__(EPlan<MODE, L, TB, REPS, CMIN, CMAX>::NWARP * 32, 1)
    qp_engine_kernel(const __grid_constant__ EngParams p) {
  using PL = EPlan<MODE, L, TB, REPS, CMIN, CMAX>;
  constexpr int NWARP = PL::NWARP;
  const int NS = p.ns;
  uint8_t* smem = qp_smem;
  if (threadIdx.x == 0 && smem_u32(qp_smem) != kDynSmemBase) __trap();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, q = lane & 3;

  TableBuild<REPS, NWARP * 32, PL::ENTRIES> tbl;
  tbl.load(p.table);

  // ---- this CTA's tiles, and this warp's share --------------------------------------------------
  const uint32_t T0 = p.cta_begin[blockIdx.x], T1 = p.cta_begin[blockIdx.x + 1];
  const uint32_t nC = T1 - T0;
  const uint32_t a = T0 + nC * warp / NWARP, b = T0 + nC * (warp + 1) / NWARP;
  // locate tile a: op oi, row tile rt, k tile kt (once per warp)
  int oi = 0;
  while (oi + 1 < p.n_ops && a >= p.op[oi + 1].tile0) ++oi;
  uint32_t rt, kt;
  {
    const uint32_t loc = a - p.op[oi].tile0;
    rt = loc / (uint32_t)p.op[oi].KT;
    kt = loc - rt * (uint32_t)p.op[oi].KT;
  }
  // ---- the code ring + its fetch cursor (runs NS tiles ahead, across layers) -------------------
  // The cursor lives in shared memory (only lane 0 issues copies), keeping the main loop's
  // register budget for the decode.
  const uint32_t ring = smem_u32(smem + PL::RING_OFF) + (uint32_t)(warp * NS * PL::STAGE);
  const uint32_t bars = smem_u32(smem + PL::BAR_OFF) + (uint32_t)(warp * NS * 8);
  struct FCur {
    const uint8_t* ptr;   // next tile to fetch
    int oi, kt;           // its layer and k tile
    uint32_t left;        // tiles left in layer oi (from ptr on)
    int pad;
  };
  static_assert(sizeof(FCur) == 24, "fetch cursor");
  FCur* fc = reinterpret_cast<FCur*>(smem + PL::BAR_OFF + 512) + warp;
  // fetch the cursor's tile into stage st and advance the cursor (lane 0)
  auto fetch = [&](int st, uint32_t dep) {
    FCur f = *fc;
    const EngOp& o = p.op[f.oi];
    const uint32_t nb = 512u * (uint32_t)(f.kt < o.KH ? o.c_lo : o.c_hi);
    const uint32_t bar = bars + 8u * st;
    mbar_expect_tx(bar, nb);
    bulk_g2s(ring + (uint32_t)(st * PL::STAGE) + dep, f.ptr, nb, bar, l2_evict_first_policy());
    f.ptr += nb;
    if (++f.kt == o.KT) f.kt = 0;
    if (--f.left == 0 && f.oi + 1 < p.n_ops) {
      ++f.oi;
      f.ptr = p.op[f.oi].codes;
      f.kt = 0;
      f.left = (uint32_t)p.op[f.oi].RT * p.op[f.oi].KT;
    }
    *fc = f;
  };
  auto init_cursor = [&]() {
    const EngOp& o = p.op[oi];
    FCur f;
    f.oi = oi;
    f.kt = (int)kt;
    f.left = (uint32_t)o.RT * o.KT - (a - o.tile0);
    f.ptr = o.codes + (long long)rt * o.rowtile_bytes +
            ((int)kt < o.KH ? (long long)kt * 512 * o.c_lo
                            : (long long)o.KH * 512 * o.c_lo + (long long)((int)kt - o.KH) * 512 * o.c_hi);
    f.pad = 0;
    *fc = f;
  };

  // ---- rotation jobs (the first CTAs): x' of every layer, before this CTA's own tiles ------------
  const bool rotor = (int)blockIdx.x < p.total_jobs;
  if (rotor) {
    asm volatile("griddepcontrol.wait;" ::: "memory");          // x may come from the previous kernel
    for (int j = blockIdx.x; j < p.total_jobs; j += gridDim.x) {
      int jo = 0;
      while (jo + 1 < p.n_ops && j >= p.op[jo + 1].job0) ++jo;
      const EngOp& o = p.op[jo];
      const int jl = j - o.job0, nblk = o.d_in / o.rht_block;
      const int beta = jl / nblk, blk = jl - beta * nblk;
      engine_rotate<NWARP>(o, p.x_dtype, beta, blk, reinterpret_cast<float*>(smem));   // table / ring area: not live
      __threadfence();
      __syncthreads();
      if (tid == 0) {
        if (atomicAdd(o.job_count, 1u) == (unsigned)(o.njobs - 1)) {   // the layer's last job: x' complete
          *o.job_count = 0u;
          __threadfence();
          atomicAdd(o.ready, 1u);
        }
      }
    }
    __syncthreads();                                            // scratch reads done before the table build
  }
  if (lane == 0) {
#pragma unroll 1
    for (int st = 0; st < NS; ++st) mbar_init(bars + 8u * st, 1);
    mbar_fence_init();
    init_cursor();
    if (a < b) fetch(0, 0u);
  }
  tbl.store(smem);
  if (lane == 0)
    for (int st = 1; st < NS && a + st < b; ++st) fetch(st, 0u);
  if (!rotor) asm volatile("griddepcontrol.wait;" ::: "memory");
  // launches of this group completed so far (stable during the launch: bumped by the last CTA out)
  const unsigned gen = ld_acquire_u32(p.gen + 1);
  __syncthreads();

  const uint32_t laneoff = (uint32_t)(lane % REPS) * 4u;
  const uint32_t mulk = (1u << (Dec<MODE, CMIN, L, TB, REPS>::KSH > 0 ? Dec<MODE, CMIN, L, TB, REPS>::KSH : 0)) + p.zero;
  const bool xrow = g < p.batch;
  // x' of op oi for this lane (row g, column group q); the wait for its rotation happens on entry
  auto enter_op = [&](int o_) {
    const EngOp& o = p.op[o_];
    if (o.njobs > 0) {
      for (;;) {
        if ((int)(ld_acquire_u32(o.ready) - (gen + 1u)) >= 0) break;
        __nanosleep(64);
      }
    }
  };
  float sc[4];
  auto load_scales = [&](int o_, uint32_t rt_) {
    const float* s = p.op[o_].scales + rt_ * kTileRows + g;
#pragma unroll
    for (int i = 0; i < 4; ++i) sc[i] = __ldg(s + 8 * i);
  };
  uint32_t xb[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) xb[i] = 0u;
  // this lane's x' row (g) and column group (q) of layer o_ (recomputed: no live register)
  auto xlane = [&](int o_) -> const __half* { return p.op[o_].xr + (size_t)g * p.op[o_].d_in + 64 * q; };
  if (a < b) {
    enter_op(oi);
    const __half* xl = xlane(oi);
    load_scales(oi, rt);
    if (xrow) {
      load_x8_coh(xb, xl + kt * kTileCols);
      load_x8_coh(xb + 8, xl + kt * kTileCols + 16);
    }
  }
  float acc[2][4];
#pragma unroll
  for (int m = 0; m < 2; ++m)
#pragma unroll
    for (int r = 0; r < 4; ++r) acc[m][r] = 0.f;
  int seg_k0 = (int)kt;
  int st = 0;
  uint32_t par = 0;
  for (uint32_t t = a; t < b; ++t) {
    const EngOp& o = p.op[oi];
    mbar_wait(bars + 8u * st, par);
    const int c = (int)kt < o.KH ? o.c_lo : o.c_hi;
    // next tile: same layer -> its first-half activations are loaded mid-tile; else on entry
    uint32_t kt_n = kt + 1, rt_n = rt;
    int oi_n = oi;
    if (kt_n == (uint32_t)o.KT) {
      kt_n = 0;
      if (++rt_n == (uint32_t)o.RT) { rt_n = 0; ++oi_n; }
    }
    const bool same_op = oi_n == oi;
    const __half* xl = xlane(oi);
    const __half* x_hi = xrow ? xl + kt * kTileCols + 32 : nullptr;
    const __half* x_next = (xrow && t + 1 < b && same_op) ? xl + kt_n * kTileCols : nullptr;
    const uint32_t src = ring + (uint32_t)(st * PL::STAGE) + (uint32_t)lane * 16u;
    c_dispatch<CMIN, CMAX>(c, [&](auto CC) {
      constexpr int C = decltype(CC)::value;
      uint32_t cur[4 * C];
#pragma unroll
      for (int i = 0; i < C; ++i) {
        const uint4 v = lds128(src + i * 512);
        cur[4 * i] = v.x; cur[4 * i + 1] = v.y; cur[4 * i + 2] = v.z; cur[4 * i + 3] = v.w;
      }
      // the stage is free once every lane's shared loads have returned (see qp_gemv_kernel)
      const uint32_t dep = __reduce_or_sync(0xffffffffu, cur[4 * C - 1] & p.zero);
      if (lane == 0 && t + NS < b) fetch(st, dep);
      tile_body<MODE, C, L, TB, REPS, false, false, true>(cur, laneoff, mulk, xb, acc, nullptr, 0, x_hi, x_next, 0u);
    });
    if (++st == NS) { st = 0; par ^= 1u; }

    if (kt == (uint32_t)o.KT - 1 || t == b - 1) {
      // ---- end of this warp's segment of row tile rt ----
      const bool own = seg_k0 == 0 && kt == (uint32_t)o.KT - 1;
      if (own) {
#pragma unroll
        for (int m = 0; m < 2; ++m)
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            const int row = 16 * m + g + 8 * (r >> 1), bb = 2 * q + (r & 1);
            if (bb < p.batch) {
              const float v = acc[m][r] * sc[2 * m + (r >> 1)];
              const size_t e = (size_t)bb * o.d_out + rt * kTileRows + row;
              if (p.y_f32) {
                float* y = reinterpret_cast<float*>(o.y) + e;
                *y = p.y_accum ? *y + v : v;
              } else {
                reinterpret_cast<__half*>(o.y)[e] = __float2half_rn(v);
              }
            }
          }
      } else {
        float* wsb = o.ws + rt * kTileRows;
#pragma unroll
        for (int m = 0; m < 2; ++m)
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            const int row = 16 * m + g + 8 * (r >> 1), bb = 2 * q + (r & 1);
            if (bb < p.batch) atomicAdd(wsb + (size_t)bb * o.d_out + row, acc[m][r] * sc[2 * m + (r >> 1)]);
          }
        const int nk = (int)kt - seg_k0 + 1;
        __threadfence();
        __syncwarp();
        int done = 0;
        if (lane == 0) done = atomicAdd(o.counters + rt, nk) + nk == o.KT;
        done = __shfl_sync(0xffffffffu, done, 0);
        if (done) {
          // every k tile of row tile rt is in the workspace: write y, re-zero the workspace
          __threadfence();
          for (int e = lane; e < kTileRows * p.batch; e += 32) {
            const int bb = e >> 5, row = e & 31;
            float* wp = wsb + (size_t)bb * o.d_out + row;
            const float v = __ldcg(wp);
            __stcg(wp, 0.f);
            const size_t ye = (size_t)bb * o.d_out + rt * kTileRows + row;
            if (p.y_f32) {
              float* y = reinterpret_cast<float*>(o.y) + ye;
              *y = p.y_accum ? *y + v : v;
            } else {
              reinterpret_cast<__half*>(o.y)[ye] = __float2half_rn(v);
            }
          }
          if (lane == 0) o.counters[rt] = 0;
        }
      }
#pragma unroll
      for (int m = 0; m < 2; ++m)
#pragma unroll
        for (int r = 0; r < 4; ++r) acc[m][r] = 0.f;
      seg_k0 = 0;
      if (t + 1 < b) {
        if (!same_op) {
          enter_op(oi_n);
          const __half* xl = xlane(oi_n);
          if (xrow) {
            load_x8_coh(xb, xl);
            load_x8_coh(xb + 8, xl + 16);
          }
        }
        load_scales(oi_n, rt_n);
      }
    }
    kt = kt_n; rt = rt_n; oi = oi_n;
  }
  asm volatile("griddepcontrol.launch_dependents;");
  // the last CTA out bumps the generation (every CTA read it at entry)
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    if (atomicAdd(p.gen, 1u) == gridDim.x - 1) {
      *p.gen = 0u;
      __threadfence();
      atomicAdd(p.gen + 1, 1u);
    }
  }
}

template <int MODE, int L, int TB, int REPS, int CMIN, int CMAX>
struct EngineVariant {
  static cudaError_t launch(const EngParams& prm0, int grid, bool pdl, cudaStream_t s) {
    using PL = EPlan<MODE, L, TB, REPS, CMIN, CMAX>;
    EngParams prm = prm0;
    prm.ns = (std::min)((std::min)(ns_cap(), 1024 / (PL::NWARP * 8)), PL::AVAIL / (PL::NWARP * PL::STAGE));
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
    auto k = qp_engine_kernel<MODE, L, TB, REPS, CMIN, CMAX>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, PL::SMEM_MAX);
    if (e == cudaSuccess) e = cudaLaunchKernelEx(&cfg, k, prm);
    return e;
  }
  static void reg() { register_engine(EngineKey{MODE, L, TB, REPS, CMIN, CMAX}, &launch); }
};

}  // namespace qp
