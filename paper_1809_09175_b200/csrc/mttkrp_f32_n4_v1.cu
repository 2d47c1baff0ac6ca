// mttkrp_f32_n4_v1.cu -- fast MTTKRP kernels for float, N = 4, 1-element lane vectors (see mttkrp.cuh).
#include "mttkrp.cuh"

namespace sptk {
SPTK_INSTANTIATE_FAST(float, 4, 1)
}  // namespace sptk
