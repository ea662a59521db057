// Micro-benchmarks that size the fused dequant-GEMV design on B200 (sm_100a).
// Not part of the product; results are recorded in profiles/ and DESIGN.md.
//   1. legacy mma.sync m16n8k16 f16->f32 issue rate per SM
//   2. mock TCQ decode (funnel shift, hash, LUT LDS, HMMA) in pairs/clk/SM for
//      a 32-replica (128 KB) and a 16-replica (64 KB) pre-signed table
//   3. mock LUT2 (VQ/NUQ) decode
//   4. streaming LDG.128 read bandwidth (the HBM ceiling for our access pattern)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ void mma16816(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
               : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
               : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__global__ void k_mma(int iters, float* out) {
  float acc[8][4] = {};
  uint32_t a[4] = {0x3c003c00u ^ threadIdx.x, 0x3c003c00u, 0x3c003c00u, 0x3c003c00u};
  uint32_t b0 = 0x3c00u, b1 = 0x3c00u;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) mma16816(acc[j], a, b0, b1);
  }
  float s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += acc[j][0] + acc[j][1] + acc[j][2] + acc[j][3];
  if (s == 12345.f) out[0] = s;
}

// S = shift bits per pair, words per trellis = 4*S.  REP32: 32-replica table (key stride 128 B)
template <int S, bool REP32, bool COMPUTE_ONLY>
__global__ void k_tcq(const uint4* __restrict__ codes, int tiles_per_warp, int ntiles, float* out) {
  extern __shared__ uint32_t tab[];
  constexpr int TABW = REP32 ? 1024 * 32 : 1024 * 16;
  for (int i = threadIdx.x; i < TABW; i += blockDim.x) tab[i] = 0x3c003c00u ^ (i * 2654435761u & 0x03ff03ffu);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const uint32_t laneoff = REP32 ? lane * 4u : (lane & 15) * 4u;
  float acc[2][4] = {};
  uint32_t xb0 = 0x3c00u + lane, xb1 = 0x3c00u;
  uint32_t w[4 * S];
  {
    const uint4* src = codes + (size_t)(gw % ntiles) * (S * 32) + lane;
#pragma unroll
    for (int c = 0; c < S; ++c) {
      uint4 v = __ldg(src + c * 32);
      w[4 * c] = v.x; w[4 * c + 1] = v.y; w[4 * c + 2] = v.z; w[4 * c + 3] = v.w;
    }
  }
  for (int t = 0; t < tiles_per_warp; ++t) {
    if (!COMPUTE_ONLY) {
      int tile = (gw * tiles_per_warp + t) % ntiles;
      const uint4* src = codes + (size_t)tile * (S * 32) + lane;
#pragma unroll
      for (int c = 0; c < S; ++c) {
        uint4 v = __ldg(src + c * 32);
        w[4 * c] = v.x; w[4 * c + 1] = v.y; w[4 * c + 2] = v.z; w[4 * c + 3] = v.w;
      }
    } else {
#pragma unroll
      for (int c = 0; c < 4 * S; ++c) w[c] = w[c] * 1664525u + t;
    }
    uint32_t a[4];
#pragma unroll
    for (int j = 0; j < 128; ++j) {
      constexpr int NW = 4 * S;
      const int o = j * S;
      const int wi = o >> 5, r = o & 31;
      uint32_t hi = w[wi], lo = w[(wi + 1) % NW];
      uint32_t win;
      if (r + 16 <= 32) win = hi >> (32 - r - 16);
      else win = __funnelshift_r(lo, hi, 64 - r - 16);
      uint32_t addr;
      if (REP32) {
        uint32_t tt = win * 2u + 2u;
        uint32_t p2 = win * tt;
        addr = (p2 & 0x1ff80u) | laneoff;
      } else {
        uint32_t p = win * win + win;
        addr = (p & 0xffc0u) | laneoff;
      }
      a[j & 3] = *reinterpret_cast<const uint32_t*>(reinterpret_cast<const char*>(tab) + addr);
      if ((j & 3) == 3) mma16816(acc[(j >> 2) & 1], a, xb0 + j, xb1);
    }
  }
  float s = acc[0][0] + acc[0][1] + acc[0][2] + acc[0][3] + acc[1][0] + acc[1][1] + acc[1][2] + acc[1][3];
  if (s == 12345.f) out[0] = s;
}

// C = index bits per pair (2b); words per run = 4*C
template <int C, bool COMPUTE_ONLY>
__global__ void k_lut2(const uint4* __restrict__ codes, int tiles_per_warp, int ntiles, float* out) {
  extern __shared__ uint32_t tab[];
  constexpr int TABW = (1 << C) * 32;
  for (int i = threadIdx.x; i < TABW; i += blockDim.x) tab[i] = 0x3c003c00u ^ (i * 2654435761u & 0x03ff03ffu);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const uint32_t laneoff = lane * 4u;
  float acc[2][4] = {};
  uint32_t xb0 = 0x3c00u + lane, xb1 = 0x3c00u;
  uint32_t w[4 * C + 1];
  {
    const uint4* src = codes + (size_t)(gw % ntiles) * (C * 32) + lane;
#pragma unroll
    for (int c = 0; c < C; ++c) {
      uint4 v = __ldg(src + c * 32);
      w[4 * c] = v.x; w[4 * c + 1] = v.y; w[4 * c + 2] = v.z; w[4 * c + 3] = v.w;
    }
    w[4 * C] = 0;
  }
  for (int t = 0; t < tiles_per_warp; ++t) {
    if (!COMPUTE_ONLY) {
      int tile = (gw * tiles_per_warp + t) % ntiles;
      const uint4* src = codes + (size_t)tile * (C * 32) + lane;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        uint4 v = __ldg(src + c * 32);
        w[4 * c] = v.x; w[4 * c + 1] = v.y; w[4 * c + 2] = v.z; w[4 * c + 3] = v.w;
      }
    } else {
#pragma unroll
      for (int c = 0; c < 4 * C; ++c) w[c] = w[c] * 1664525u + t;
    }
    uint32_t a[4];
#pragma unroll
    for (int j = 0; j < 128; ++j) {
      const int o = j * C;
      const int wi = o >> 5, r = o & 31;
      // field occupies MSB-first bits [r, r+C) of (w[wi]:w[wi+1]); put its LSB at bit 7
      uint32_t f = __funnelshift_r(w[wi + 1], w[wi], 57 - r - C > 31 ? 31 : 57 - r - C);
      if (57 - r - C > 31) f = w[wi] >> (57 - r - C - 32);
      uint32_t addr = (f & (((1u << C) - 1) << 7)) | laneoff;
      a[j & 3] = *reinterpret_cast<const uint32_t*>(reinterpret_cast<const char*>(tab) + addr);
      if ((j & 3) == 3) mma16816(acc[(j >> 2) & 1], a, xb0 + j, xb1);
    }
  }
  float s = acc[0][0] + acc[0][1] + acc[0][2] + acc[0][3] + acc[1][0] + acc[1][1] + acc[1][2] + acc[1][3];
  if (s == 12345.f) out[0] = s;
}

__global__ void k_stream(const uint4* __restrict__ src, size_t n16, uint32_t* out) {
  uint32_t x = 0;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n16; i += 4 * stride) {
    uint4 a = __ldg(src + i), b = __ldg(src + i + stride), c = __ldg(src + i + 2 * stride), d = __ldg(src + i + 3 * stride);
    x ^= a.x ^ a.y ^ a.z ^ a.w ^ b.x ^ b.y ^ b.z ^ b.w ^ c.x ^ c.y ^ c.z ^ c.w ^ d.x ^ d.y ^ d.z ^ d.w;
  }
  for (; i < n16; i += stride) { uint4 a = __ldg(src + i); x ^= a.x ^ a.y ^ a.z ^ a.w; }
  if (x == 0x12345678u) out[0] = x;
}

__global__ void k_clock(unsigned long long* out) {
  unsigned long long t0 = clock64();
  unsigned long long g0; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  unsigned long long g1 = g0;
  while (g1 - g0 < 2000000ull) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = g1 - g0; }
}

template <typename F>
float time_it(F f, int reps) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  f();
  cudaDeviceSynchronize();
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  return ms / reps;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  const int nsm = p.multiProcessorCount;
  printf("device %s sms=%d l2=%d MB smem/blk optin=%zu\n", p.name, nsm, p.l2CacheSize >> 20, p.sharedMemPerBlockOptin);
  float* out; CK(cudaMalloc(&out, 64));
  unsigned long long* clk; CK(cudaMalloc(&clk, 16));
  k_clock<<<nsm, 32>>>(clk);
  CK(cudaDeviceSynchronize());
  unsigned long long hc[2]; cudaMemcpy(hc, clk, 16, cudaMemcpyDeviceToHost);
  double ghz = (double)hc[0] / hc[1];
  printf("sm clock (idle-ish, spin) %.3f GHz\n", ghz);

  // 1. mma
  for (int warps : {4, 8, 16}) {
    int iters = 2000;
    float ms = time_it([&] { k_mma<<<nsm, warps * 32>>>(iters, out); }, 5);
    double mmas = (double)nsm * warps * iters * 8;
    double tflops = mmas * 4096 / (ms * 1e-3) / 1e12;
    printf("mma.sync m16n8k16 f32acc: warps/SM=%d  %.1f TFLOP/s  (%.2f HMMA/clk/SM at %.2f GHz)\n", warps, tflops,
           mmas / nsm / (ms * 1e-3) / (ghz * 1e9), ghz);
  }
  // 4. stream
  size_t nbytes = (size_t)4 << 30;
  uint4* big; CK(cudaMalloc(&big, nbytes));
  CK(cudaMemset(big, 1, nbytes));
  for (int bl : {2, 4, 8}) {
    float ms = time_it([&] { k_stream<<<nsm * bl, 512>>>(big, nbytes / 16, (uint32_t*)out); }, 5);
    printf("stream LDG.128 read  blocks/SM=%d: %.1f GB/s\n", bl, nbytes / (ms * 1e-3) / 1e9);
  }
  // 2/3. decode mocks over a 1 GB code buffer (no L2 reuse)
  auto run_tcq = [&](auto kern, int S, int tabbytes, int warps, const char* name) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, tabbytes);
    int tile_bytes = 512 * S;
    int ntiles = (int)(((size_t)1 << 30) / tile_bytes);
    int tpw = ntiles / (nsm * warps);
    float ms = time_it([&] { kern<<<nsm, warps * 32, tabbytes>>>(big, tpw, ntiles, out); }, 3);
    cudaError_t e = cudaGetLastError(); if (e != cudaSuccess) { printf("%s warps=%d: launch error %s\n", name, warps, cudaGetErrorString(e)); return; }
    double pairs = (double)nsm * warps * tpw * 4096;
    double bytes = (double)nsm * warps * tpw * tile_bytes;
    printf("%s warps=%d: %.2f pairs/clk/SM  %.1f GB/s codes  (%.1f%% of 6535)\n", name, warps,
           pairs / nsm / (ms * 1e-3) / (ghz * 1e9), bytes / (ms * 1e-3) / 1e9, 100 * bytes / (ms * 1e-3) / 6535e9);
  };
  for (int warps : {4, 8, 16}) {
    run_tcq(k_tcq<4, true, true>, 4, 131072, warps, "COMPUTE tcq s=4 rep32");
    run_tcq(k_tcq<4, false, true>, 4, 65536, warps, "COMPUTE tcq s=4 rep16");
    run_tcq(k_tcq<5, true, true>, 5, 131072, warps, "COMPUTE tcq s=5 rep32");
    run_tcq(k_tcq<8, true, true>, 8, 131072, warps, "COMPUTE tcq s=8 rep32");
    run_tcq(k_lut2<4, true>, 4, 16 * 128, warps, "COMPUTE lut2 c=4");
    run_tcq(k_lut2<6, true>, 6, 64 * 128, warps, "COMPUTE lut2 c=6");
    run_tcq(k_lut2<8, true>, 8, 256 * 128, warps, "COMPUTE lut2 c=8");
  }
  for (int warps : {16, 32}) {
    run_tcq(k_tcq<5, true, false>, 5, 131072, warps, "LOAD tcq s=5 rep32");
    run_tcq(k_lut2<6, false>, 6, 64 * 128, warps, "LOAD lut2 c=6");
  }
  CK(cudaDeviceSynchronize());
  cudaMemcpy(hc, clk, 16, cudaMemcpyDeviceToHost);
  return 0;
}
