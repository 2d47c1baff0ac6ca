// mttkrp_generic.cu -- generic MTTKRP kernels (any N <= 6, any R; see mttkrp.cuh).
#include "mttkrp.cuh"

namespace sptk {

template <typename T>
sptk_status launch_generic(int G, const MttkrpArgs &a, int64_t workers, cudaStream_t s) {
    const int64_t threads = workers * G;
    const unsigned blocks = (unsigned)((threads + 255) / 256);
    if (G == 4) launch_pdl(mttkrp_generic_kernel<T, 4, 4>, blocks, 256, 0, s, a);
    else launch_pdl(mttkrp_generic_kernel<T, 32, 4>, blocks, 256, 0, s, a);
    count_launch();
    SPTK_CUDA(cudaGetLastError());
    return SPTK_OK;
}

template sptk_status launch_generic<double>(int, const MttkrpArgs &, int64_t, cudaStream_t);
template sptk_status launch_generic<float>(int, const MttkrpArgs &, int64_t, cudaStream_t);

}  // namespace sptk
