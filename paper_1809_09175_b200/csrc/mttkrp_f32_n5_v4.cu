// mttkrp_f32_n5_v4.cu -- fast MTTKRP kernels for float, N = 5, 4-element lane vectors (see mttkrp.cuh).
#include "mttkrp.cuh"

namespace sptk {
SPTK_INSTANTIATE_FAST(float, 5, 4)
}  // namespace sptk
