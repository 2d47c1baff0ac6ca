// mttkrp_f32_n4_v4.cu -- fast MTTKRP kernels for float, N = 4, 4-element lane vectors (see mttkrp.cuh).
#include "mttkrp.cuh"

namespace sptk {
SPTK_INSTANTIATE_FAST(float, 4, 4)
}  // namespace sptk
