// LDS throughput vs address pattern on sm_100a (32-bit loads, conflict-free banks)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int ROWBITS, int MODE>
__global__ void k_lds(int iters, uint32_t* out) {
  extern __shared__ uint32_t tab[];
  constexpr int WORDS = (1 << ROWBITS) * 32;
  for (int i = threadIdx.x; i < WORDS; i += blockDim.x) tab[i] = i * 2654435761u;
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31;
  uint32_t x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = (threadIdx.x * 7919u + k * 104729u);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      uint32_t row;
      if (MODE == 0) row = 0;                       // same row, distinct banks
      else if (MODE == 1) row = (x[k] >> 7);        // random rows, distinct banks (bank = lane)
      else row = (x[k] >> 7);                       // random rows, random banks
      uint32_t addr = ((row & ((1u << ROWBITS) - 1)) << 7) | (MODE == 2 ? (x[k] & 0x7c) : lane * 4);
      x[k] += *reinterpret_cast<const uint32_t*>(reinterpret_cast<const char*>(tab) + addr);
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s ^= x[k];
  if (s == 0x1234567u) out[0] = s;
}
template <typename K>
void run(K k, int rowbits, const char* name, int nsm, uint32_t* out) {
  int smem = (1 << rowbits) * 128;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int iters = 4000;
  for (int warps : {8, 16, 32}) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    k<<<nsm, warps * 32, smem>>>(iters, out);
    cudaEventRecord(a);
    k<<<nsm, warps * 32, smem>>>(iters, out);
    cudaEventRecord(b); cudaEventSynchronize(b);
    cudaError_t e = cudaGetLastError();
    float ms; cudaEventElapsedTime(&ms, a, b);
    double lds = (double)warps * iters * 8;   // per SM
    printf("%-28s rowbits=%2d warps=%2d: %.3f LDS(warp)/clk/SM %s\n", name, rowbits, warps, lds / (ms * 1e-3) / 1.965e9,
           e == cudaSuccess ? "" : cudaGetErrorString(e));
  }
}
int main() {
  uint32_t* out; cudaMalloc(&out, 64);
  int nsm = 148;
  run(k_lds<4, 0>, 4, "same-row", nsm, out);
  run(k_lds<4, 1>, 4, "rand-row bank=lane", nsm, out);
  run(k_lds<8, 1>, 8, "rand-row bank=lane", nsm, out);
  run(k_lds<10, 1>, 10, "rand-row bank=lane", nsm, out);
  run(k_lds<10, 2>, 10, "rand-row rand-bank", nsm, out);
  return 0;
}
