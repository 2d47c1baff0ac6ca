// mttkrp_f64_n5_v1.cu -- fast MTTKRP kernels for double, N = 5, 1-element lane vectors (see mttkrp.cuh).
#include "mttkrp.cuh"

namespace sptk {
SPTK_INSTANTIATE_FAST(double, 5, 1)
}  // namespace sptk
