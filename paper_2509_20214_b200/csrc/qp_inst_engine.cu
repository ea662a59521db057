// Persistent multi-layer engine variants (qp_engine.cuh). One variant per decode-table family;
// the TCQ variants take every step width c in [CMIN, CMAX] at run time.
#include "qp_engine.cuh"

namespace qp {
namespace {
struct Register {
  Register() {
    EngineVariant<DEC_TCQ_PRESIGNED, 16, 9, 32, 5, 8>::reg();    // TCQ 2.5-4.0, half-TCQ 2.75-3.75 (C2)
    EngineVariant<DEC_TCQ_PRESIGNED, 16, 9, 32, 3, 4>::reg();    // TCQ 1.5-2.0, half-TCQ 1.75
    EngineVariant<DEC_TCQ_PRESIGNED, 16, 9, 32, 4, 5>::reg();    // half-TCQ 2.25
    EngineVariant<DEC_TCQ_UNSIGNED, 16, 10, 32, 8, 9>::reg();    // TCQ 4.5, half-TCQ 4.25
    EngineVariant<DEC_LUT2, 0, 0, 32, 4, 4>::reg();              // VQ 2.0, NUQ / UNIF 2
    EngineVariant<DEC_LUT2, 0, 0, 32, 5, 5>::reg();              // VQ 2.5
    EngineVariant<DEC_LUT2, 0, 0, 32, 6, 6>::reg();              // VQ 3.0, NUQ / UNIF 3
    EngineVariant<DEC_LUT2, 0, 0, 32, 7, 7>::reg();              // VQ 3.5
    EngineVariant<DEC_LUT2, 0, 0, 32, 8, 8>::reg();              // VQ 4.0, NUQ / UNIF 4
    EngineVariant<DEC_LUT2, 0, 0, 32, 9, 9>::reg();              // VQ 4.5
  }
} register_instance;
}  // namespace

// experiment builds (-DQP_ENG_TIMELINE): copy the per-CTA stamps of the last engine launch
extern "C" int qp_debug_engine_timeline(unsigned long long* host, int n) {
#ifdef QP_ENG_TIMELINE
  if (n > kMaxEngCtas * 24) n = kMaxEngCtas * 24;
  const int n1 = n < kMaxEngCtas * 8 ? n : kMaxEngCtas * 8;
  cudaError_t e = cudaMemcpyFromSymbol(host, g_eng_tl, (size_t)n1 * 8);
  if (e == cudaSuccess && n > n1) e = cudaMemcpyFromSymbol(host + n1, g_eng_wl, (size_t)(n - n1) * 8);
  return (int)e;
#else
  (void)host;
  (void)n;
  return -1;
#endif
}
}  // namespace qp
