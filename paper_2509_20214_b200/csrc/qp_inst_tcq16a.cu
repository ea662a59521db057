// Kernel variants compiled in this unit (generated list; see qp_gemv.cuh).
#include "qp_gemv.cuh"

namespace qp {
namespace {
struct Register {
  Register() {
    GemvVariant<DEC_TCQ_PRESIGNED, 3, 3, 16, 9, 32>::reg();
    GemvVariant<DEC_TCQ_PRESIGNED, 4, 4, 16, 9, 32>::reg();
    GemvVariant<DEC_TCQ_PRESIGNED, 5, 5, 16, 9, 32, true>::reg();
    GemvVariant<DEC_TCQ_PRESIGNED, 6, 6, 16, 9, 32>::reg();
  }
} register_instance;
}  // namespace
}  // namespace qp
