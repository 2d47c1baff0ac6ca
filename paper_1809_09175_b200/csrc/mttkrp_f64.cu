// mttkrp_f64.cu -- instantiations of the MTTKRP kernels for double (see mttkrp.cuh).
#include "mttkrp.cuh"

namespace sptk {

template <typename T, int N, int RB, int U, bool SORTED>
static sptk_status fast_g(int G, const MttkrpArgs &a, int64_t workers, cudaStream_t s) {
    const int64_t threads = workers * G;
    const unsigned blocks = (unsigned)((threads + 255) / 256);
    switch (G) {
    case 1: mttkrp_fast_kernel<T, N, 1, U, RB, SORTED><<<blocks, 256, 0, s>>>(a); break;
    case 2: mttkrp_fast_kernel<T, N, 2, U, RB, SORTED><<<blocks, 256, 0, s>>>(a); break;
    case 4: mttkrp_fast_kernel<T, N, 4, U, RB, SORTED><<<blocks, 256, 0, s>>>(a); break;
    case 8: mttkrp_fast_kernel<T, N, 8, U, RB, SORTED><<<blocks, 256, 0, s>>>(a); break;
    case 16: mttkrp_fast_kernel<T, N, 16, U, RB, SORTED><<<blocks, 256, 0, s>>>(a); break;
    case 32: mttkrp_fast_kernel<T, N, 32, U, RB, SORTED><<<blocks, 256, 0, s>>>(a); break;
    default: return fail(SPTK_EINVAL, "fast MTTKRP: bad lane count");
    }
    count_launch();
    SPTK_CUDA(cudaGetLastError());
    return SPTK_OK;
}

template <typename T, bool SORTED>
static sptk_status fast_n(int N, int G, int rb, const MttkrpArgs &a, int64_t workers,
                          cudaStream_t s) {
    constexpr int U = 2;
    switch (N) {
    case 3:
        if constexpr (sizeof(T) == 4)
            if (rb == 16) return fast_g<T, 3, 16, U, SORTED>(G, a, workers, s);
        return fast_g<T, 3, 32, U, SORTED>(G, a, workers, s);
    case 4: return fast_g<T, 4, 32, U, SORTED>(G, a, workers, s);
    case 5: return fast_g<T, 5, 32, U, SORTED>(G, a, workers, s);
    default: return fail(SPTK_EINVAL, "fast MTTKRP: N must be 3..5");
    }
}

template <>
sptk_status launch_fast<double>(int N, int G, int rb, const MttkrpArgs &a, int64_t workers,
                             cudaStream_t s) {
    return a.perm ? fast_n<double, false>(N, G, rb, a, workers, s)
                  : fast_n<double, true>(N, G, rb, a, workers, s);
}

template <>
sptk_status launch_generic<double>(int G, const MttkrpArgs &a, int64_t workers, cudaStream_t s) {
    const int64_t threads = workers * G;
    const unsigned blocks = (unsigned)((threads + 255) / 256);
    if (G == 4) mttkrp_generic_kernel<double, 4, 4><<<blocks, 256, 0, s>>>(a);
    else mttkrp_generic_kernel<double, 32, 4><<<blocks, 256, 0, s>>>(a);
    count_launch();
    SPTK_CUDA(cudaGetLastError());
    return SPTK_OK;
}

}  // namespace sptk
