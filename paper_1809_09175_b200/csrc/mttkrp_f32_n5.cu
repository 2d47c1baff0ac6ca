// mttkrp_f32_n5.cu -- fast MTTKRP kernels for float, N = 5 (see mttkrp.cuh).
#include "mttkrp.cuh"

namespace sptk {
SPTK_INSTANTIATE_FAST(float, 5)
}  // namespace sptk
