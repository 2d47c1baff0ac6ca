// mttkrp_f64_n3.cu -- fast MTTKRP kernels for double, N = 3 (see mttkrp.cuh).
#include "mttkrp.cuh"

namespace sptk {
SPTK_INSTANTIATE_FAST(double, 3)
}  // namespace sptk
