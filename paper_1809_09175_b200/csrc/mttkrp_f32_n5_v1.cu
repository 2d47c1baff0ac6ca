// mttkrp_f32_n5_v1.cu -- fast MTTKRP kernels for float, N = 5, 1-element lane vectors (see mttkrp.cuh).
#include "mttkrp.cuh"

namespace sptk {
SPTK_INSTANTIATE_FAST(float, 5, 1)
}  // namespace sptk
