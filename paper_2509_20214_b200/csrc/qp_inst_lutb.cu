// Kernel variants compiled in this unit (generated list; see qp_gemv.cuh).
#include "qp_gemv.cuh"

namespace qp {
namespace {
struct Register {
  Register() {
    GemvVariant<DEC_LUT2, 8, 8, 0, 0, 32>::reg();
    GemvVariant<DEC_LUT2, 9, 9, 0, 0, 32>::reg();
    GemvVariant<DEC_LUT2, 10, 10, 0, 0, 32>::reg();
    GemvVariant<DEC_LUT2, 11, 11, 0, 0, 16>::reg();
    GemvVariant<DEC_LUT2, 12, 12, 0, 0, 8>::reg();
  }
} register_instance;
}  // namespace
}  // namespace qp
