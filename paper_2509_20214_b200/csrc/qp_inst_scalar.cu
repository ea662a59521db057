// Kernel variants compiled in this unit (generated list; see qp_gemv.cuh).
#include "qp_gemv.cuh"

namespace qp {
namespace {
struct Register {
  Register() {
    GemvVariant<DEC_SCALAR, 10, 10, 0, 5, 32>::reg();
    GemvVariant<DEC_SCALAR, 12, 12, 0, 6, 32>::reg();
    GemvVariant<DEC_SCALAR, 14, 14, 0, 7, 32>::reg();
    GemvVariant<DEC_SCALAR, 16, 16, 0, 8, 32>::reg();
  }
} register_instance;
}  // namespace
}  // namespace qp
