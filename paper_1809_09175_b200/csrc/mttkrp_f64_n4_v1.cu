// mttkrp_f64_n4_v1.cu -- fast MTTKRP kernels for double, N = 4, 1-element lane vectors (see mttkrp.cuh).
#include "mttkrp.cuh"

namespace sptk {
SPTK_INSTANTIATE_FAST(double, 4, 1)
}  // namespace sptk
