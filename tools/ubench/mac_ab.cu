// Where should the multiply-accumulate of the fused dequant-GEMV run on B200? ("make a
// measured tcgen05 decision", "add the hfma2 CUDA-core comparison".)
//
// The decode of the real kernel (TCQ: funnel-shift window, (w+1)w hash, key shift, mask | lane, LDS
// from the 32-replica 128 KB table; register-resident streams, no HBM) feeding four MAC variants,
// 148 CTAs x 16 warps, pairs / clk / SM (SM clock measured on the box):
//   HMMA    mma.sync m16n8k16 f16 -> f32, one per 4 pairs per lane (the product)
//   NONE    no MAC (XOR-accumulate): the upper bound of any MAC offload
//   HFMA2   CUDA cores, batch 1: one HFMA2 per pair (half2 accumulators, flushed to fp32 per k-step)
//           -- the paper's "CC" kernels
//   TC05x1  each decoded A fragment (4 regs = one m16 x k16 block) stored to tensor memory with
//           tcgen05.st.16x256b.x1 (the layout of an mma.sync A fragment), tcgen05.wait::st per tile:
//           the data movement a tcgen05.mma path with A in TMEM would add in place of the HMMAs
//           (the MMAs themselves are issued by one thread per 128-row group, not per warp)
//   TC05x2  the same with two fragments per tcgen05.st (16x256b.x2)
// Not part of the product; results: profiles/r2/mac_ab.txt, DESIGN.md section 8.
#include <cstdint>
#include <cstdio>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

enum { HMMA = 0, NONE = 1, HFMA2 = 2, TC05X1 = 3, TC05X2 = 4 };

__device__ __forceinline__ void mma16816(float* c, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
               : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3]) : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t lds(uint32_t off) {
  uint32_t v;
  asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(off));
  return v;
}
__device__ __forceinline__ void tst_x1(uint32_t taddr, uint32_t r0, uint32_t r1, uint32_t r2, uint32_t r3) {
  asm volatile("tcgen05.st.sync.aligned.16x256b.x1.b32 [%0], {%1, %2, %3, %4};" :: "r"(taddr), "r"(r0), "r"(r1), "r"(r2), "r"(r3) : "memory");
}
__device__ __forceinline__ void tst_x2(uint32_t taddr, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.16x256b.x2.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};"
               :: "r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]) : "memory");
}

template <int S, int V>
__global__ void __launch_bounds__(512, 1) k(int iters, float* out, uint32_t seed) {
  extern __shared__ __align__(1024) uint8_t tab[];
  __shared__ uint32_t tmem_base;
  for (int i = threadIdx.x; i < 32768; i += blockDim.x) reinterpret_cast<uint32_t*>(tab)[i] = 0x3c003c00u ^ (i * 2654435761u & 0x03ff03ffu);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (V == TC05X1 || V == TC05X2) {
    if (warp == 0) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"((uint32_t)__cvta_generic_to_shared(&tmem_base)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
  }
  __syncthreads();
  if (V == TC05X1 || V == TC05X2) asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tbase = (V == TC05X1 || V == TC05X2) ? tmem_base : 0u;
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(tab);
  const uint32_t laneoff = base + lane * 4u;
  float acc[2][4] = {};
  float facc[4] = {};
  uint32_t xacc = 0;
  constexpr int NW = 4 * S;
  uint32_t w[NW];
#pragma unroll
  for (int c = 0; c < NW; ++c) w[c] = seed * (threadIdx.x + 7 * c + 1);
  const uint32_t xb0 = 0x3c00u + lane, xb1 = 0x3c00u;
  const __half2 xh = __halves2half2(__ushort_as_half(0x3c00), __ushort_as_half((unsigned short)(0x3800 + lane)));
  // this warp's TMEM lanes: 32 * (warp % 4); the 4 warp-groups of the CTA own column quarters
  const uint32_t lane_base = (uint32_t)(32 * (warp & 3)) << 16;
  const uint32_t col0 = (uint32_t)(128 * (warp >> 2));
  for (int t = 0; t < iters; ++t) {
#pragma unroll
    for (int c = 0; c < NW; ++c) w[c] ^= t;
    uint32_t a[16];
    __half2 hacc = __float2half2_rn(0.f);
#pragma unroll
    for (int j = 0; j < 128; ++j) {
      const int o = j * S;
      const int wi = (o >> 5) % NW, r = o & 31;
      const uint32_t hi = w[wi], lo = w[(wi + 1) % NW];
      uint32_t win;
      if (r + 16 <= 32) win = hi >> (32 - r - 16);
      else win = __funnelshift_r(lo, hi, 64 - r - 16);
      const uint32_t p = win * win + win;
      const uint32_t addr = ((p + p) & 0x1ff80u) | laneoff;
      const uint32_t v = lds(addr);
      if (V == HFMA2) {
        hacc = __hfma2(*reinterpret_cast<const __half2*>(&v), xh, hacc);
        if ((j & 7) == 7) {           // per k-step: half2 partial -> fp32
          const float2 f = __half22float2(hacc);
          facc[(j >> 3) & 3] += f.x + f.y;
          hacc = __float2half2_rn(0.f);
        }
        continue;
      }
      a[j & 15] = v;
      const int i0 = (j & 15) - 3;
      if ((j & 3) == 3) {
        const int kap = j >> 3, m = (j >> 2) & 1;
        if (V == NONE) xacc ^= a[i0] ^ a[i0 + 1] ^ a[i0 + 2] ^ a[i0 + 3];
        else if (V == HMMA) mma16816(acc[m], a[i0], a[i0 + 1], a[i0 + 2], a[i0 + 3], xb0, xb1);
        else if (V == TC05X1)   // A fragment (a0 a1 a2 a3) -> 16x256b register order (a0 a2 a1 a3)
          tst_x1(tbase + lane_base + ((uint32_t)(16 * m) << 16) + col0 + 8 * kap, a[i0], a[i0 + 2], a[i0 + 1], a[i0 + 3]);
      }
      if (V == TC05X2 && (j & 15) == 15) {   // k-steps kap-1, kap of each m block: one store per m
        const int kap = j >> 3;
#pragma unroll
        for (int m = 0; m < 2; ++m) {
          uint32_t r8[8] = {a[4 * m], a[4 * m + 2], a[4 * m + 1], a[4 * m + 3],
                            a[8 + 4 * m], a[8 + 4 * m + 2], a[8 + 4 * m + 1], a[8 + 4 * m + 3]};
          tst_x2(tbase + lane_base + ((uint32_t)(16 * m) << 16) + col0 + 8 * (kap - 1), r8);
        }
      }
    }
    if (V == TC05X1 || V == TC05X2) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  float s = acc[0][0] + acc[0][1] + acc[0][2] + acc[0][3] + acc[1][0] + acc[1][1] + acc[1][2] + acc[1][3] + (float)xacc +
            facc[0] + facc[1] + facc[2] + facc[3];
  if (s == 12345.f) out[0] = s;
  if (V == TC05X1 || V == TC05X2) {
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(tbase));
  }
}

__global__ void k_clock(unsigned long long* out) {
  unsigned long long t0 = clock64(), g0, g1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  g1 = g0;
  while (g1 - g0 < 5000000ull) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) { out[0] = t1 - t0; out[1] = g1 - g0; }
}

template <int S, int V>
int run(const char* name, double ghz) {
  float* out; CK(cudaMalloc(&out, 64));
  auto f = k<S, V>;
  CK(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072 + 1024));
  f<<<148, 512, 131072 + 1024>>>(4, out, 3);
  CK(cudaDeviceSynchronize());
  const int iters = 400;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  f<<<148, 512, 131072 + 1024>>>(iters, out, 3);
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms; cudaEventElapsedTime(&ms, a, b);
  const double pairs = 148.0 * 16 * 32 * iters * 128;
  printf("%-8s s=%d 16 warps  %6.2f pairs/clk/SM  (%.3f ms, %.3f GHz)\n", name, S, pairs / (ms * 1e-3 * ghz * 1e9) / 148, ms, ghz);
  cudaFree(out);
  return 0;
}

int main() {
  unsigned long long* c; CK(cudaMalloc(&c, 16));
  k_clock<<<148, 32>>>(c);
  CK(cudaDeviceSynchronize());
  unsigned long long h[2]; cudaMemcpy(h, c, 16, cudaMemcpyDeviceToHost);
  const double ghz = (double)h[0] / h[1];
  for (int rep = 0; rep < 2; ++rep) {
    run<5, HMMA>("HMMA", ghz);
    run<5, NONE>("NONE", ghz);
    run<5, HFMA2>("HFMA2", ghz);
    run<5, TC05X1>("TC05x1", ghz);
    run<5, TC05X2>("TC05x2", ghz);
    run<8, HMMA>("HMMA", ghz);
    run<8, NONE>("NONE", ghz);
    run<8, TC05X1>("TC05x1", ghz);
  }
  return 0;
}
