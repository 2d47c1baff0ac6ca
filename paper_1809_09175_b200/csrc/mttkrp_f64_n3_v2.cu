// mttkrp_f64_n3_v2.cu -- fast MTTKRP kernels for double, N = 3, 2-element lane vectors (see mttkrp.cuh).
#include "mttkrp.cuh"

namespace sptk {
SPTK_INSTANTIATE_FAST(double, 3, 2)
}  // namespace sptk
