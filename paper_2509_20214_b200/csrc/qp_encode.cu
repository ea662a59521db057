// GPU tail-biting trellis encoder: the rotate-half Viterbi of
// qp_quantize_offline (reading R4) for many trellises at once.
//
// One CTA encodes one trellis (T = 256 weights, n = 128 steps of V = 2) at a time:
//   pass 1: v rolled by n/2 steps, free start, free end (argmin, lowest index); trace back to the
//           state S at the original wrap boundary (rolled step n - n/2 - 1);
//   pass 2: the unrolled v with start state = end state = S; trace back to the windows.
// DP step i (P:1049 windows, LAYOUT.md bit order): for every new state sigma' (the low L-s bits of
// a window) and every k < 2^s, the window w = k 2^(L-s) + sigma' costs D[w >> s] + ||v_i - LUT[w]||^2;
// the new D[sigma'] is the minimum, ties to the lowest k (reading R5). LUT[w] is the hybrid
// codeword of P:1025-1033: p = (w+1) w mod 2^L, sign = bit L-1, idx = bits [L-tb-1, L-2].
// Arithmetic is float64 with explicitly rounded operations in the host encoder's order, so the
// windows are bitwise those of the host encoder (qp_offline.cpp Viterbi::run).
#include <cuda_runtime.h>

#include <cstdint>

#include "qp_internal.h"

namespace qp {

namespace {

constexpr int kEncThreads = 512;
constexpr int kSteps = 128;   // n = T / V

struct EncParams {
  const double* v;        // [units][128][2] standardized weights in LAYOUT.md step order
  int units;
  int L, s, tb;
  const double* tlut;     // [2^tb][2]
  uint32_t* windows;      // [units][128]
  uint16_t* bp;           // [gridDim.x][128][2^(L-s)] backpointers (k of the best predecessor)
};

__device__ __forceinline__ void lut_value(const double* tl, uint32_t w, int L, int tb, double& a, double& b) {
  const uint32_t mask = L >= 32 ? 0xffffffffu : ((1u << L) - 1u);
  const uint32_t p = (uint32_t)(((unsigned long long)(w + 1) * w) & mask);
  const bool neg = (p >> (L - 1)) & 1u;
  const uint32_t idx = (p >> (L - tb - 1)) & ((1u << tb) - 1u);
  a = neg ? -tl[2 * idx] : tl[2 * idx];
  b = tl[2 * idx + 1];
}

// one Viterbi pass over v (rolled by `roll` steps); start / end < 0: free. Leaves the windows of
// the best path in win[0..127] (shared). Returns nothing: the caller reads win.
__device__ void viterbi_pass(const EncParams& p, const double* v, int roll, int start, int end, double* D, double* Dn,
                             const double* tl, uint16_t* bp, uint32_t* win, double* red_v, int* red_i) {
  const int L = p.L, s = p.s, ns = 1 << (L - s), nk = 1 << s;
  const int tid = threadIdx.x;
  const double inf = __longlong_as_double(0x7ff0000000000000ll);
  for (int i = tid; i < ns; i += kEncThreads) D[i] = (start < 0 || i == start) ? 0.0 : inf;
  __syncthreads();
  for (int i = 0; i < kSteps; ++i) {
    const int src = (i + roll) % kSteps;
    const double v0 = v[2 * src], v1 = v[2 * src + 1];
    uint16_t* bpi = bp + (size_t)i * ns;
    for (int sp = tid; sp < ns; sp += kEncThreads) {
      double best = inf;
      int bk = 0;
      for (int k = 0; k < nk; ++k) {
        const uint32_t w = (uint32_t)(k * ns + sp);
        double t0, t1;
        lut_value(tl, w, L, p.tb, t0, t1);
        const double d0 = __dsub_rn(v0, t0), d1 = __dsub_rn(v1, t1);
        const double c = __dadd_rn(D[w >> s], __dadd_rn(__dmul_rn(d0, d0), __dmul_rn(d1, d1)));
        if (c < best) {
          best = c;
          bk = k;
        }
      }
      Dn[sp] = best;
      bpi[sp] = (uint16_t)bk;
    }
    __syncthreads();
    double* t = D;
    D = Dn;
    Dn = t;
  }
  // end state: given, or the argmin (lowest index on ties)
  int sig = end;
  if (sig < 0) {
    double bv = inf;
    int bi = ns;
    for (int i = tid; i < ns; i += kEncThreads)
      if (D[i] < bv) {   // ascending i per thread: the first minimum
        bv = D[i];
        bi = i;
      }
    red_v[tid] = bv;
    red_i[tid] = bi;
    __syncthreads();
    for (int h = kEncThreads / 2; h > 0; h >>= 1) {
      if (tid < h) {
        const double ov = red_v[tid + h];
        const int oi = red_i[tid + h];
        if (ov < red_v[tid] || (ov == red_v[tid] && oi < red_i[tid])) {
          red_v[tid] = ov;
          red_i[tid] = oi;
        }
      }
      __syncthreads();
    }
    sig = red_i[0];
    if (sig >= ns) sig = 0;        // every state infinite (cannot happen for finite inputs)
  }
  __syncthreads();
  if (tid == 0) {
    __threadfence_block();
    for (int i = kSteps - 1; i >= 0; --i) {
      const int k = bp[(size_t)i * ns + sig];
      const uint32_t w = (uint32_t)(k * ns + sig);
      win[i] = w;
      sig = (int)(w >> s);
    }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kEncThreads, 1) qp_tcq_viterbi_kernel(const __grid_constant__ EncParams p) {
  extern __shared__ __align__(16) uint8_t sm[];
  const int ns = 1 << (p.L - p.s), ntl = 1 << p.tb;
  double* D = reinterpret_cast<double*>(sm);
  double* Dn = D + ns;
  double* tl = Dn + ns;
  double* v = tl + 2 * ntl;
  double* red_v = v + 2 * kSteps;
  int* red_i = reinterpret_cast<int*>(red_v + kEncThreads);
  uint32_t* win = reinterpret_cast<uint32_t*>(red_i + kEncThreads);
  for (int i = threadIdx.x; i < 2 * ntl; i += kEncThreads) tl[i] = p.tlut[i];
  uint16_t* bp = p.bp + (size_t)blockIdx.x * kSteps * ns;
  for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
    __syncthreads();
    for (int i = threadIdx.x; i < 2 * kSteps; i += kEncThreads) v[i] = p.v[(size_t)u * 2 * kSteps + i];
    __syncthreads();
    // pass 1: rolled by n/2, free start and end; S = the state after rolled step n - n/2 - 1
    const int h = kSteps / 2;
    viterbi_pass(p, v, h, -1, -1, D, Dn, tl, bp, win, red_v, red_i);
    const int S = (int)(win[kSteps - h - 1] & (uint32_t)(ns - 1));
    __syncthreads();
    // pass 2: unrolled, start = end = S
    viterbi_pass(p, v, 0, S, S, D, Dn, tl, bp, win, red_v, red_i);
    for (int i = threadIdx.x; i < kSteps; i += kEncThreads) p.windows[(size_t)u * kSteps + i] = win[i];
  }
}

}  // namespace

size_t tcq_viterbi_scratch_bytes(int L, int s, int grid) {
  return (size_t)grid * kSteps * ((size_t)1 << (L - s)) * sizeof(uint16_t);
}

// Encode `units` trellises (v: device [units][128][2] float64) into their windows (device
// [units][128]). bp_scratch: tcq_viterbi_scratch_bytes(L, s, grid) bytes. Synchronous errors only.
cudaError_t launch_tcq_viterbi(const double* v, int units, int L, int s, int tb, const double* tlut_dev,
                               uint32_t* windows, uint16_t* bp_scratch, int grid, cudaStream_t st) {
  EncParams p{};
  p.v = v;
  p.units = units;
  p.L = L;
  p.s = s;
  p.tb = tb;
  p.tlut = tlut_dev;
  p.windows = windows;
  p.bp = bp_scratch;
  const int ns = 1 << (L - s), ntl = 1 << tb;
  const size_t smem = (size_t)(2 * ns + 2 * ntl + 2 * kSteps + kEncThreads) * sizeof(double) +
                      (size_t)kEncThreads * sizeof(int) + (size_t)kSteps * sizeof(uint32_t);
  cudaError_t e = cudaFuncSetAttribute(qp_tcq_viterbi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  qp_tcq_viterbi_kernel<<<grid, kEncThreads, smem, st>>>(p);
  count_launch();
  return cudaGetLastError();
}

}  // namespace qp
