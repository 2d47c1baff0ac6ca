// mttkrp_atomic.cu -- the paper's atomic-per-nonzero MTTKRP (VerA/VerB,
// Figs. mttkrp_alg / mttkrp_array; SURVEY §8(f)
// NEXT-1): nonzeros in STORAGE order, every nonzero's row contribution added
// to V with atomics ("Multiple teams may be contributing to the same entries",
// hence the atomic add).  No permutation is needed (the
// zero-preprocessing path).  Same B200 lane mapping as the permuted
// kernels (a group of G lanes spans R, 32-byte vector rows), so the contrast
// with sptk_mttkrp is the traversal and the write discipline only.
#include "mttkrp.cuh"

namespace sptk {

// vector columns: lane q owns V = 32/sizeof(T) consecutive columns of the tile
template <typename T, int G>
__global__ void __launch_bounds__(256) mttkrp_atomic_vec_kernel(const MttkrpArgs a) {
    constexpr int V = 32 / sizeof(T);
    const int64_t gtid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t worker = gtid / G;
    const int q = (int)(gtid % G);
    const int64_t s = a.pos_begin + worker * a.run;
    if (s >= a.pos_end) return;
    const int64_t e = min(s + a.run, a.pos_end);
    if (q * V >= a.ncols) return;
    const int c = a.col0 + q * V;
    const int off = sizeof(T) / 4;
    T lam[V];
#pragma unroll
    for (int v = 0; v < V; ++v) lam[v] = T(1);
    if (a.lambda) ld_row(static_cast<const T *>(a.lambda) + c, lam);
    T *__restrict__ out = static_cast<T *>(a.out);
    for (int64_t i = s; i < e; ++i) {
        const uint8_t *r = a.rec + (size_t)i * a.rb;
        const uint32_t *ix = reinterpret_cast<const uint32_t *>(r) + off;
        const T x = __ldg(reinterpret_cast<const T *>(r));
        T t[V];
#pragma unroll
        for (int v = 0; v < V; ++v) t[v] = x * lam[v];
#pragma unroll
        for (int m = 0; m < kMaxModes; ++m) {
            if (m >= a.N || m == a.mode) continue;
            T f[V];
            ld_row(static_cast<const T *>(a.A[m]) + (int64_t)__ldg(ix + m) * a.ld + c, f);
#pragma unroll
            for (int v = 0; v < V; ++v) t[v] *= f[v];
        }
        red_row(out + (int64_t)__ldg(ix + a.mode) * a.ld + c, t);
    }
}

// scalar columns (any R, any alignment): lane q owns columns col0 + q + 32k
template <typename T>
__global__ void __launch_bounds__(256) mttkrp_atomic_scalar_kernel(const MttkrpArgs a) {
    constexpr int G = 32, NV = 4;
    const int64_t gtid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t worker = gtid / G;
    const int q = (int)(gtid % G);
    const int64_t s = a.pos_begin + worker * a.run;
    if (s >= a.pos_end) return;
    const int64_t e = min(s + a.run, a.pos_end);
    const int off = sizeof(T) / 4;
    T *__restrict__ out = static_cast<T *>(a.out);
    for (int64_t i = s; i < e; ++i) {
        const uint8_t *r = a.rec + (size_t)i * a.rb;
        const uint32_t *ix = reinterpret_cast<const uint32_t *>(r) + off;
        const T x = __ldg(reinterpret_cast<const T *>(r));
        const int64_t row = __ldg(ix + a.mode);
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            const int j = q + G * k;
            if (j >= a.ncols) break;
            const int col = a.col0 + j;
            T t = a.lambda ? x * static_cast<const T *>(a.lambda)[col] : x;
            for (int m = 0; m < a.N; ++m)
                if (m != a.mode) t *= __ldg(static_cast<const T *>(a.A[m]) + (int64_t)__ldg(ix + m) * a.ld + col);
            atomicAdd(out + row * a.ld + col, t);
        }
    }
}

template <typename T>
static sptk_status launch_atomic(sptk_tensor t, MttkrpArgs &a, int64_t R, bool vec,
                                 cudaStream_t s) {
    constexpr int V = 32 / sizeof(T);
    a.run = 16;
    const int64_t workers = (t->P + a.run - 1) / a.run;
    if (vec) {
        const int64_t tile = 32 * V;
        for (int64_t c0 = 0; c0 < R; c0 += tile) {
            a.col0 = (int)c0;
            a.ncols = (int)((R - c0) < tile ? (R - c0) : tile);
            int G = 1;
            while (G * V < a.ncols) G <<= 1;
            const unsigned blocks = (unsigned)((workers * G + 255) / 256);
            switch (G) {
            case 1: mttkrp_atomic_vec_kernel<T, 1><<<blocks, 256, 0, s>>>(a); break;
            case 2: mttkrp_atomic_vec_kernel<T, 2><<<blocks, 256, 0, s>>>(a); break;
            case 4: mttkrp_atomic_vec_kernel<T, 4><<<blocks, 256, 0, s>>>(a); break;
            case 8: mttkrp_atomic_vec_kernel<T, 8><<<blocks, 256, 0, s>>>(a); break;
            case 16: mttkrp_atomic_vec_kernel<T, 16><<<blocks, 256, 0, s>>>(a); break;
            default: mttkrp_atomic_vec_kernel<T, 32><<<blocks, 256, 0, s>>>(a); break;
            }
            count_launch();
            SPTK_CUDA(cudaGetLastError());
        }
    } else {
        for (int64_t c0 = 0; c0 < R; c0 += 128) {
            a.col0 = (int)c0;
            a.ncols = (int)((R - c0) < 128 ? (R - c0) : 128);
            const unsigned blocks = (unsigned)((workers * 32 + 255) / 256);
            mttkrp_atomic_scalar_kernel<T><<<blocks, 256, 0, s>>>(a);
            count_launch();
            SPTK_CUDA(cudaGetLastError());
        }
    }
    return SPTK_OK;
}

}  // namespace sptk

using namespace sptk;

extern "C" sptk_status sptk_mttkrp_atomic(sptk_tensor t, int mode, int64_t R,
                                          const void *const *factors, const void *lambda,
                                          void *out, void *stream) {
    if (!t) return fail(SPTK_EINVAL, "null tensor handle");
    if (t->poisoned) return fail(SPTK_ECUDA, "tensor handle poisoned by an earlier CUDA error");
    if (mode < 0 || mode >= t->N) return fail(SPTK_EINVAL, "mode out of range");
    if (R < 1 || R > (int64_t(1) << 20)) return fail(SPTK_EINVAL, "R must be in [1, 2^20]");
    if (!factors || !out) return fail(SPTK_EINVAL, "factors/out is NULL");
    for (int m = 0; m < t->N; ++m)
        if (m != mode && !factors[m]) return fail(SPTK_EINVAL, "factors[m] is NULL");
    if (t->deterministic)
        return fail(SPTK_EUNSUPPORTED, "the atomic-per-nonzero MTTKRP is not deterministic");
    cudaStream_t s = (cudaStream_t)stream;
    const size_t es = dtype_bytes(t->dtype);
    sptk_status st = SPTK_OK;
    if (cudaMemsetAsync(out, 0, (size_t)t->dims[mode] * R * es, s) != cudaSuccess)
        st = cuda_fail(cudaGetLastError(), "memset out");
    if (st == SPTK_OK && t->P > 0) {
        MttkrpArgs a{};
        a.rec = t->rec.as<uint8_t>();
        a.pos_begin = 0;
        a.pos_end = t->P;
        a.ld = R;
        a.mode = mode;
        a.N = t->N;
        a.rb = t->rec_bytes;
        for (int m = 0; m < t->N; ++m) a.A[m] = (m == mode) ? nullptr : factors[m];
        a.lambda = lambda;
        a.out = out;
        const int V = 32 / (int)es;
        auto al = [](const void *p) { return (reinterpret_cast<uintptr_t>(p) & 31) == 0; };
        bool vec = R % V == 0 && al(out) && (!lambda || al(lambda));
        for (int m = 0; m < t->N && vec; ++m)
            if (m != mode && !al(factors[m])) vec = false;
        set_dispatch(vec ? "atomic V" + std::to_string(V) : std::string("atomic V1"));
        cudaEvent_t ev;
        st = mttkrp_span_begin(s, &ev);
        if (st == SPTK_OK)
            st = t->dtype == SPTK_F64 ? launch_atomic<double>(t, a, R, vec, s)
                                      : launch_atomic<float>(t, a, R, vec, s);
        if (st == SPTK_OK) st = mttkrp_span_end(s, ev);
    }
    if (st == SPTK_ECUDA) t->poisoned = true;
    return st;
}
