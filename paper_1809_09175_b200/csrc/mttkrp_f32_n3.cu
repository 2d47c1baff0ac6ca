// mttkrp_f32_n3.cu -- fast MTTKRP kernels for float, N = 3 (see mttkrp.cuh).
#include "mttkrp.cuh"

namespace sptk {
SPTK_INSTANTIATE_FAST(float, 3)
}  // namespace sptk
