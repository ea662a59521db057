// Micro-benchmark of the fused dequant-GEMV prologue on B200: cost of building the 128 KB
// 32-way replicated decode table in shared memory, per CTA (clock64) and per launch (events).
// Not part of the product; results go to profiles/.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int NT = 512;
constexpr int TAB = 131072;

template <int MODE>   // 0 empty, 1 STS only, 2 LDG+STS, 3 LDG only, 4 STS.32 loop, 5 LDG(16 copies)+STS
__global__ void __launch_bounds__(NT, 1) k(const uint32_t* __restrict__ g, unsigned long long* t, float* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  unsigned long long t0 = clock64();
  constexpr int B = TAB / 16 / NT;  // 16
  uint32_t v[B];
  if (MODE == 5) {
#pragma unroll
    for (int i = 0; i < B; ++i) v[i] = __ldg(g + (blockIdx.x % 16) * 1024 + (threadIdx.x + i * NT) / 8);
  } else if (MODE == 2 || MODE == 3) {
#pragma unroll
    for (int i = 0; i < B; ++i) v[i] = __ldg(g + (threadIdx.x + i * NT) / 8);
  } else {
#pragma unroll
    for (int i = 0; i < B; ++i) v[i] = threadIdx.x * 7 + i;
  }
  if (MODE == 1 || MODE == 2 || MODE == 5) {
#pragma unroll
    for (int i = 0; i < B; ++i)
      *reinterpret_cast<uint4*>(sm + (size_t)(threadIdx.x + i * NT) * 16) = make_uint4(v[i], v[i], v[i], v[i]);
  }
  if (MODE == 3) {
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < B; ++i) s ^= v[i];
    if (s == 0x12345678u) out[0] = 1.f;
  }
  if (MODE == 4) {
    for (int i = threadIdx.x; i < TAB / 4; i += NT) reinterpret_cast<uint32_t*>(sm)[i] = v[i & 15];
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) { t[blockIdx.x * 2] = t0; t[blockIdx.x * 2 + 1] = t1; }
  if (sm[threadIdx.x * 4] == 0xAB && threadIdx.x == 9999) out[1] = 1.f;
}

template <int MODE>
int run(const char* name, const uint32_t* g, unsigned long long* t, float* out, int smem) {
  CK(cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  cudaStream_t s; CK(cudaStreamCreate(&s));
  for (int i = 0; i < 5; ++i) k<MODE><<<148, NT, smem, s>>>(g, t, out);
  CK(cudaStreamSynchronize(s));
  cudaGraph_t gr; cudaGraphExec_t ge;
  CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal));
  for (int i = 0; i < 40; ++i) k<MODE><<<148, NT, smem, s>>>(g, t, out);
  CK(cudaStreamEndCapture(s, &gr));
  CK(cudaGraphInstantiate(&ge, gr, 0));
  CK(cudaGraphLaunch(ge, s));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a, s);
  for (int r = 0; r < 10; ++r) CK(cudaGraphLaunch(ge, s));
  cudaEventRecord(b, s);
  CK(cudaEventSynchronize(b));
  float ms; cudaEventElapsedTime(&ms, a, b);
  unsigned long long h[296];
  CK(cudaMemcpy(h, t, sizeof h, cudaMemcpyDeviceToHost));
  double cyc = 0, mx = 0;
  for (int i = 0; i < 148; ++i) { double d = (double)(h[2 * i + 1] - h[2 * i]); cyc += d; if (d > mx) mx = d; }
  printf("%-28s smem=%6d  per-CTA %7.0f cyc (max %7.0f)   per launch %6.2f us\n", name, smem, cyc / 148, mx,
         ms * 1e3 / 400);
  return 0;
}

int main() {
  uint32_t* g; unsigned long long* t; float* out;
  CK(cudaMalloc(&g, 16 * 4096 * 4)); CK(cudaMemset(g, 1, 16 * 4096 * 4));
  CK(cudaMalloc(&t, 296 * 8)); CK(cudaMalloc(&out, 64));
  for (int smem : {1024, 140000, 217000}) {
    run<0>("empty", g, t, out, smem);
  }
  run<1>("STS.128 x16 (128 KB)", g, t, out, 217000);
  run<2>("LDG x16 + STS.128 x16", g, t, out, 217000);
  run<3>("LDG x16 only", g, t, out, 217000);
  run<4>("STS.32 loop (128 KB)", g, t, out, 217000);
  run<5>("LDG(16 copies) + STS.128", g, t, out, 217000);
  return 0;
}
