// Kernel variants compiled in this unit (generated list; see qp_gemv.cuh).
#include "qp_gemv.cuh"

namespace qp {
namespace {
struct Register {
  Register() {
    GemvVariant<DEC_TCQ_PRESIGNED, 7, 7, 16, 9, 32>::reg();
    GemvVariant<DEC_TCQ_PRESIGNED, 8, 8, 16, 9, 32, true>::reg();
    GemvVariant<DEC_TCQ_UNSIGNED, 9, 9, 16, 10, 32>::reg();
    GemvVariant<DEC_TCQ_UNSIGNED, 10, 10, 16, 11, 16>::reg();
  }
} register_instance;
}  // namespace
}  // namespace qp
