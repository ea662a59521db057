// Kernel variants compiled in this unit (generated list; see qp_gemv.cuh).
#include "qp_gemv.cuh"

namespace qp {
namespace {
struct Register {
  Register() {
    GemvVariant<DEC_LUT2, 3, 3, 0, 0, 32>::reg();
    GemvVariant<DEC_LUT2, 4, 4, 0, 0, 32>::reg();
    GemvVariant<DEC_LUT2, 5, 5, 0, 0, 32>::reg();
    GemvVariant<DEC_LUT2, 6, 6, 0, 0, 32>::reg();
    GemvVariant<DEC_LUT2, 7, 7, 0, 0, 32>::reg();
  }
} register_instance;
}  // namespace
}  // namespace qp
