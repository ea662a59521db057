// Randomized Hadamard rotation of the activations, x' = (1/sqrt(b)) blockdiag(H_b) D x
// (P:345-349), plus small utility kernels and the variant registry.
//
// One CTA per (block of b inputs, batch row). Each thread holds E consecutive elements:
// log2(E) butterfly stages in registers, up to 5 stages across lanes with shfl.xor, the
// remaining stages through shared memory. fp32 arithmetic, one RNE rounding to fp16.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cstdlib>
#include <mutex>
#include <vector>

#include "qp_internal.h"

namespace qp {

// Zero the fp32 outputs the next GEMV accumulates into (grid-stride over all CTAs).
__device__ __forceinline__ void zero_outputs(const RhtParams& p) {
  const long long nthr = (long long)gridDim.x * gridDim.y * blockDim.x;
  const long long me = ((long long)blockIdx.y * gridDim.x + blockIdx.x) * blockDim.x + threadIdx.x;
  for (int i = 0; i < p.n_zero; ++i) {
    float4* z = reinterpret_cast<float4*>(p.zero_ptr[i]);
    const long long n4 = p.zero_n[i] / 4;
    for (long long j = me; j < n4; j += nthr) z[j] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (long long j = n4 * 4 + me; j < p.zero_n[i]; j += nthr) p.zero_ptr[i][j] = 0.f;
  }
}

__global__ void qp_zero_kernel(const __grid_constant__ RhtParams p) {
  asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  zero_outputs(p);
}

template <int E>
__global__ void __launch_bounds__(1024) qp_rht_kernel(const __grid_constant__ RhtParams p) {
  extern __shared__ float sx[];
  const int blk = blockIdx.x, beta = blockIdx.y;
  const int nthr = p.block / E;
  const int t = threadIdx.x;
  const int base = blk * p.block + t * E;     // global input index of v[0]
  float v[E];
  // Let the dependent GEMV start its prologue (code prefetch, decode-table build) right away;
  // it waits for this grid's completion before it reads x' or touches y.
  asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  zero_outputs(p);
  const size_t row = (size_t)beta * p.d_in;
  if (p.x_dtype == 0) {
    const __half* x = reinterpret_cast<const __half*>(p.x) + row + base;
#pragma unroll
    for (int i = 0; i < E; i += 8) {
      const uint4 u = *reinterpret_cast<const uint4*>(x + i);
      const __half2* h = reinterpret_cast<const __half2*>(&u);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float2 f = __half22float2(h[k]);
        v[i + 2 * k] = f.x;
        v[i + 2 * k + 1] = f.y;
      }
    }
  } else if (p.x_dtype == 1) {
    const __nv_bfloat16* x = reinterpret_cast<const __nv_bfloat16*>(p.x) + row + base;
#pragma unroll
    for (int i = 0; i < E; ++i) v[i] = __bfloat162float(x[i]);
  } else {
    const float* x = reinterpret_cast<const float*>(p.x) + row + base;
#pragma unroll
    for (int i = 0; i < E; i += 4) {
      const float4 f = *reinterpret_cast<const float4*>(x + i);
      v[i] = f.x; v[i + 1] = f.y; v[i + 2] = f.z; v[i + 3] = f.w;
    }
  }
  // D: sign bits (1 = negative), E <= 32 consecutive bits starting at `base`
#pragma unroll
  for (int i = 0; i < E; ++i) {
    const int idx = base + i;
    if ((__ldg(p.signs + (idx >> 5)) >> (idx & 31)) & 1u) v[i] = -v[i];
  }
  // stages inside the thread: strides 1 .. E/2
#pragma unroll
  for (int h = 1; h < E; h <<= 1) {
#pragma unroll
    for (int i = 0; i < E; ++i) {
      if ((i & h) == 0) {
        const float a = v[i], b = v[i + h];
        v[i] = a + b;
        v[i + h] = a - b;
      }
    }
  }
  // stages across lanes: stride E*m, m = 1..16 (partner thread t ^ m)
  const int lane = t & 31;
  for (int m = 1; m < 32 && m < nthr; m <<= 1) {
    const bool upper = (lane & m) != 0;
#pragma unroll
    for (int i = 0; i < E; ++i) {
      const float o = __shfl_xor_sync(0xffffffffu, v[i], m);
      v[i] = upper ? (o - v[i]) : (v[i] + o);
    }
  }
  // stages across warps through shared memory: strides 32E .. block/2
  for (int h = 32 * E; h < p.block; h <<= 1) {
    __syncthreads();
#pragma unroll
    for (int i = 0; i < E; ++i) sx[t * E + i] = v[i];
    __syncthreads();
#pragma unroll
    for (int i = 0; i < E; ++i) {
      const int k = t * E + i;
      const float o = sx[k ^ h];
      v[i] = (k & h) ? (o - v[i]) : (v[i] + o);
    }
  }
  __half* out = p.out + row + base;
#pragma unroll
  for (int i = 0; i < E; i += 8) {
    uint4 u;
    __half2* h = reinterpret_cast<__half2*>(&u);
#pragma unroll
    for (int k = 0; k < 4; ++k) h[k] = __floats2half2_rn(v[i + 2 * k] * p.scale, v[i + 2 * k + 1] * p.scale);
    *reinterpret_cast<uint4*>(out + i) = u;
  }
  (void)nthr;
}

cudaError_t launch_rht(const RhtParams& p, bool pdl, cudaStream_t s) {
  int E = 8;
  while (p.block / E > 1024) E *= 2;
  if (E > 32 || p.block / E < 32) return cudaErrorInvalidValue;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.d_in / p.block, p.batch);
  cfg.blockDim = dim3(p.block / E);
  cfg.dynamicSmemBytes = p.block > 32 * E ? p.block * sizeof(float) : 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e;
  if (E == 8) {
    e = cudaFuncSetAttribute(qp_rht_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cfg.dynamicSmemBytes);
    if (e == cudaSuccess) e = cudaLaunchKernelEx(&cfg, qp_rht_kernel<8>, p);
  } else if (E == 16) {
    e = cudaFuncSetAttribute(qp_rht_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cfg.dynamicSmemBytes);
    if (e == cudaSuccess) e = cudaLaunchKernelEx(&cfg, qp_rht_kernel<16>, p);
  } else {
    e = cudaFuncSetAttribute(qp_rht_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cfg.dynamicSmemBytes);
    if (e == cudaSuccess) e = cudaLaunchKernelEx(&cfg, qp_rht_kernel<32>, p);
  }
  if (e == cudaSuccess) count_launch();
  return e;
}

cudaError_t launch_zero(const RhtParams& p, int grid, bool pdl, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(1024);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, qp_zero_kernel, p);
  if (e == cudaSuccess) count_launch();
  return e;
}

// [world][batch][m] (all-gather output) -> [batch][world*m]
__global__ void qp_gather_permute_kernel(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst, int world,
                                         int batch, int m, int eb) {
  const long long n = (long long)world * batch * m;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / ((long long)batch * m);
    const long long rem = i - r * batch * m;
    const long long b = rem / m, j = rem - b * m;
    const long long o = b * (long long)world * m + r * m + j;
    for (int k = 0; k < eb; ++k) dst[o * eb + k] = src[i * eb + k];
  }
}

// Spin-wait guard of the cross-rank waits: a peer that never arrives (a crashed or mismatched rank)
// traps after ~20 s instead of hanging the GPU; the host sees QP_ERR_CUDA on a later call.
__device__ __forceinline__ unsigned long long gtimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
constexpr unsigned long long kPeerTimeoutNs = 20ull * 1000 * 1000 * 1000;

// Fused all-gather completion on this rank: flags_local[q] counts the launches rank q has
// completed into our y_full; flags_local[world] is how many we have consumed. Waits until every
// rank is one ahead, then consumes (graph-replay safe: no host-side epoch).
__global__ void qp_peer_wait_kernel(unsigned* flags_local, int world, int n) {
  if (threadIdx.x != 0) return;
  const unsigned want = flags_local[world] + (unsigned)n;   // n deliveries per rank this round
  const unsigned long long t0 = gtimer_ns();
  for (int q = 0; q < world; ++q) {
    unsigned v;
    for (;;) {
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flags_local + q) : "memory");
      if ((int)(v - want) >= 0) break;
      if (gtimer_ns() - t0 > kPeerTimeoutNs) __trap();
      __nanosleep(64);
    }
  }
  flags_local[world] = want;
  __threadfence_system();
}


// Start of a fused all-gather round on this rank: announce to every peer that this rank has entered
// round n (so its readers of round n-1's y_full, earlier on its stream, are done): bump
// flag_peers[k][world + 1 + rank]; then wait until every peer has entered round n too
// (flags_local[world + 1 + k] >= flags_local[world] + 1, the rounds this rank has consumed + 1).
// Only then may this rank store round n into the peers' y_full.
__global__ void qp_peer_enter_kernel(PeerFlags f) {
  if (threadIdx.x != 0) return;
  const int world = f.world;
  for (int k = 0; k < world; ++k) atomicAdd_system(f.peers[k] + world + 1 + f.rank, 1u);
  __threadfence_system();
  unsigned* local = f.peers[f.rank];
  const unsigned want = local[world] + 1u;
  const unsigned long long t0 = gtimer_ns();
  for (int k = 0; k < world; ++k) {
    unsigned v;
    for (;;) {
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(local + world + 1 + k) : "memory");
      if ((int)(v - want) >= 0) break;
      if (gtimer_ns() - t0 > kPeerTimeoutNs) __trap();
      __nanosleep(64);
    }
  }
}

cudaError_t launch_peer_enter(unsigned* const* flag_peers, int rank, int world, cudaStream_t s) {
  PeerFlags f{};
  f.world = world;
  f.rank = rank;
  for (int k = 0; k < world; ++k) f.peers[k] = flag_peers[k];
  qp_peer_enter_kernel<<<1, 32, 0, s>>>(f);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_peer_wait(unsigned* flags_local, int world, cudaStream_t s, int n) {
  qp_peer_wait_kernel<<<1, 32, 0, s>>>(flags_local, world, n);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_gather_permute(const void* src, void* dst, int world, int batch, int m, int eb, cudaStream_t s) {
  const long long n = (long long)world * batch * m;
  int grid = (int)((n + 255) / 256);
  if (grid > 4096) grid = 4096;
  qp_gather_permute_kernel<<<grid, 256, 0, s>>>(static_cast<const uint8_t*>(src), static_cast<uint8_t*>(dst), world,
                                                 batch, m, eb);
  count_launch();
  return cudaGetLastError();
}

int fused_rht_max_rounds() {
  // in-CTA rotation rounds (each: an L2 round trip for x + the butterflies) above which the
  // separate, PDL-overlapped rotation kernel is cheaper (profiles/r1/ab_xs_r1.md section 5)
  static int n = -1;
  if (n < 0) {
    const char* e = getenv("QP_FUSED_RHT_ROUNDS");
    n = e ? atoi(e) : 4;
  }
  return n;
}

int ns_cap() {
  // 2 stages per warp keep the codes NS tiles ahead and leave the rest of shared memory to L1,
  // where the activations stay resident: up to 12% faster than 3-4 stages for the small-table
  // schemes, whose rings would otherwise take all of it (profiles/r1/ab_xs_r1.md section 15)
  static int n = -1;
  if (n < 0) {
    const char* e = getenv("QP_NS_MAX");
    n = e ? atoi(e) : 2;
    if (n < 1) n = 1;
    if (n > 4) n = 4;   // the mbarrier area holds 16 warps x 4 stages (1024 B)
  }
  return n;
}

int rp2_min_batch() {
  // smallest batch for the row-pair GEMV units (QP_RP2_MIN_BATCH; profiles/r1/ab_xs_r1.md section 9)
  static int n = -1;
  if (n < 0) {
    const char* e = getenv("QP_RP2_MIN_BATCH");
    n = e ? atoi(e) : 8;
  }
  return n;
}

int env_no_xs() {
  // x' staged in shared memory is opt-in (QP_XS=1): measured slower than the register path on
  // the C2 shapes (profiles/r1/ab_xs_r1.md)
  static int n = -1;
  if (n < 0) {
    const char* e = getenv("QP_XS");
    n = (e && atoi(e) != 0) ? 0 : 1;
  }
  return n;
}

// ---- variant registry ----------------------------------------------------------------
namespace {
struct Entry {
  KernelKey k;
  GemvLauncher f;
};
std::vector<Entry>& registry() {
  static std::vector<Entry> r;
  return r;
}
std::mutex& registry_mu() {
  static std::mutex m;
  return m;
}
}  // namespace

void register_gemv(const KernelKey& k, GemvLauncher f) {
  std::lock_guard<std::mutex> g(registry_mu());
  registry().push_back({k, f});
}

GemvLauncher find_gemv(const KernelKey& k) {
  std::lock_guard<std::mutex> g(registry_mu());
  for (const auto& e : registry())
    if (e.k == k) return e.f;
  return nullptr;
}

namespace {
struct EngEntry {
  EngineKey k;
  EngineLauncher f;
};
std::vector<EngEntry>& eng_registry() {
  static std::vector<EngEntry> r;
  return r;
}
}  // namespace

void register_engine(const EngineKey& k, EngineLauncher f) {
  std::lock_guard<std::mutex> g(registry_mu());
  eng_registry().push_back({k, f});
}

EngineLauncher find_engine(int mode, int L, int tb, int reps, int cmin, int cmax) {
  std::lock_guard<std::mutex> g(registry_mu());
  const EngEntry* best = nullptr;
  for (const auto& e : eng_registry())
    if (e.k.mode == mode && e.k.L == L && e.k.tb == tb && e.k.reps == reps && e.k.cmin <= cmin && e.k.cmax >= cmax &&
        (!best || e.k.cmax - e.k.cmin < best->k.cmax - best->k.cmin))
      best = &e;
  return best ? best->f : nullptr;
}

}  // namespace qp
