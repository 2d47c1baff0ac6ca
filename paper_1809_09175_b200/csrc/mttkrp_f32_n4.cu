// mttkrp_f32_n4.cu -- fast MTTKRP kernels for float, N = 4 (see mttkrp.cuh).
#include "mttkrp.cuh"

namespace sptk {
SPTK_INSTANTIATE_FAST(float, 4)
}  // namespace sptk
