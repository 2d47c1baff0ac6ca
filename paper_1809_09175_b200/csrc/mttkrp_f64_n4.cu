// mttkrp_f64_n4.cu -- fast MTTKRP kernels for double, N = 4 (see mttkrp.cuh).
#include "mttkrp.cuh"

namespace sptk {
SPTK_INSTANTIATE_FAST(double, 4)
}  // namespace sptk
