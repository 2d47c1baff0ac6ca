// mttkrp_f32_n3_v1.cu -- fast MTTKRP kernels for float, N = 3, 1-element lane vectors (see mttkrp.cuh).
#include "mttkrp.cuh"

namespace sptk {
SPTK_INSTANTIATE_FAST(float, 3, 1)
}  // namespace sptk
