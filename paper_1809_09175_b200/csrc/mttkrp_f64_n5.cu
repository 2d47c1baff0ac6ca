// mttkrp_f64_n5.cu -- fast MTTKRP kernels for double, N = 5 (see mttkrp.cuh).
#include "mttkrp.cuh"

namespace sptk {
SPTK_INSTANTIATE_FAST(double, 5)
}  // namespace sptk
