// mttkrp_f32_n3_v4.cu -- fast MTTKRP kernels for float, N = 3, 4-element lane vectors (see mttkrp.cuh).
#include "mttkrp.cuh"

namespace sptk {
SPTK_INSTANTIATE_FAST(float, 3, 4)
}  // namespace sptk
