// Issue/pipe throughput of the integer ops in the TCQ decode step on B200 (sm_100a):
// warp-instructions per clock per SM for IMAD (multiply), IMAD.IADD-style x+x, SHF, LOP3, IADD3,
// and the decode mix. 8 independent chains per thread, 16 warps per SM, 148 CTAs.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

template <int OP>
__global__ void k(int iters, uint32_t seed, uint32_t* out) {
  uint32_t v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = seed * (threadIdx.x + 1) + i * 0x9E3779B9u;
  uint32_t s1 = seed | 1u, s2 = seed ^ 0x55u;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (OP == 0) v[i] = v[i] * v[i] + v[i];                                  // IMAD (mul)
        if (OP == 1) asm volatile("add.u32 %0, %0, %0;" : "+r"(v[i]));           // x + x
        if (OP == 2) asm volatile("shf.r.wrap.b32 %0, %0, %1, 5;" : "+r"(v[i]) : "r"(s1));   // SHF
        if (OP == 3) v[i] = (v[i] & 0x1ff80u) | s2;                              // LOP3
        if (OP == 4) asm volatile("add.u32 %0, %0, %1;" : "+r"(v[i]) : "r"(s1));  // IADD
        if (OP == 5) asm volatile("mul.lo.u32 %0, %0, %1;" : "+r"(v[i]) : "r"(s1));  // IMUL
        if (OP == 6) asm volatile("shl.b32 %0, %0, 1;" : "+r"(v[i]));            // shl 1
        if (OP == 7) asm volatile("mad.lo.u32 %0, %0, 2, %1;" : "+r"(v[i]) : "r"(s2));  // IMAD imm
      }
    }
  }
  uint32_t x = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) x ^= v[i];
  if (x == 0x12345u) out[0] = x;
}

template <int OP>
int run(const char* name) {
  uint32_t* out; CK(cudaMalloc(&out, 64));
  const int iters = 2000;
  k<OP><<<148, 512>>>(10, 3, out);
  CK(cudaDeviceSynchronize());
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  k<OP><<<148, 512>>>(iters, 3, out);
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms; cudaEventElapsedTime(&ms, a, b);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double winst = 148.0 * 16 * iters * 16 * 8;      // warp instructions (approx, 1 per op)
  const double cyc = ms * 1e-3 * 1.9e9;                    // assume ~1.9 GHz under load
  printf("%-22s %.3f warp-instr/clk/SM (at 1.9 GHz)   %.2f ms\n", name, winst / cyc / 148, ms);
  cudaFree(out);
  return 0;
}

int main() {
  run<0>("IMAD w*w+w");
  run<1>("add x+x");
  run<2>("SHF.R.W");
  run<3>("LOP3 and|or");
  run<4>("IADD");
  run<5>("IMUL lo");
  run<6>("SHL 1");
  run<7>("IMAD x*2+c (imm)");
  return 0;
}
