// pack.cu -- ingest: validate 0 <= l_im < I_m
// (Eq. (2) index domain, P:147 with 0-based code P:225), convert to uint32
// and write packed AoS records {value, idx[N], pad} of 16 or 32 bytes, so a
// permuted access to nonzero p is a single aligned 16/32-byte load (§5 P:516:
// "nonzeros are ... accessed in a more random fashion").  Also produces
// ||X||^2 = sum x_i^2 (cached for the CP-ALS fit) with a deterministic
// two-stage reduction.  When memory allows, the same pass also emits every
// mode's sort keys as uint32[N][P] (the conclusion's "sorting ... while the
// tensor is being read"): build_perm's radix sorts then start from
// them instead of re-reading the 16/32-byte records once per mode.
#include "common.cuh"

namespace sptk {

sptk_status launch_sum_f64(const double *in, int64_t n, double *out, cudaStream_t s);

// idx/vals hold nonzeros [pos0, pos0 + P) of the tensor (a chunk; pos0 = 0
// and P = nnz for a device-resident input); keys are laid out for Ptot nonzeros.
template <typename T, typename I, int RB>
__global__ void __launch_bounds__(256) pack_kernel(const I *__restrict__ idx,
                                                   const T *__restrict__ vals, int64_t P,
                                                   int64_t pos0, int64_t Ptot, int N,
                                                   const int64_t *__restrict__ dims_unused,
                                                   uint64_t d0, uint64_t d1, uint64_t d2,
                                                   uint64_t d3, uint64_t d4, uint64_t d5,
                                                   uint8_t *__restrict__ rec,
                                                   uint32_t *__restrict__ keys, int *flag,
                                                   double *__restrict__ partial) {
    const uint64_t dims[6] = {d0, d1, d2, d3, d4, d5};
    double sq = 0.0;
    int bad = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P;
         i += (int64_t)gridDim.x * blockDim.x) {
        uint32_t w[RB / 4];
#pragma unroll
        for (int k = 0; k < RB / 4; ++k) w[k] = 0;
        const T x = vals[i];
        if constexpr (sizeof(T) == 8) {
            const uint64_t b = __double_as_longlong((double)x);
            w[0] = (uint32_t)b;
            w[1] = (uint32_t)(b >> 32);
        } else {
            w[0] = __float_as_uint((float)x);
        }
        const int off = sizeof(T) / 4;
#pragma unroll
        for (int m = 0; m < kMaxModes; ++m) {
            if (m < N) {
                const int64_t c = (int64_t)idx[i * N + m];
                if (c < 0 || (uint64_t)c >= dims[m]) bad = 1;
                if (off + m < RB / 4) w[off + m] = (uint32_t)c;
                if (keys) keys[(size_t)m * Ptot + pos0 + i] = (uint32_t)c;
            }
        }
        uint4 *dst = reinterpret_cast<uint4 *>(rec + (size_t)(pos0 + i) * RB);
        dst[0] = make_uint4(w[0], w[1], w[2], w[3]);
        if constexpr (RB == 32) dst[1] = make_uint4(w[4], w[5], w[6], w[7]);
        const double xd = (double)x;
        sq += xd * xd;
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
    // block reduction of sq (fixed order) -> partial[blockIdx.x]
    __shared__ double sh[256];
    sh[threadIdx.x] = sq;
    __syncthreads();
    for (int s = 128; s > 0; s >>= 1) {
        if ((int)threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x == 0) partial[blockIdx.x] = sh[0];
}

template <typename T, typename I>
static void pack_dispatch(sptk_tensor t, const void *idx, const void *vals, int64_t P, int64_t off,
                          int *flag, double *partial, int blocks, cudaStream_t s) {
    const int64_t *d = t->dims;
    auto dm = [&](int m) { return m < t->N ? (uint64_t)d[m] : (uint64_t)0; };
    if (t->rec_bytes == 16)
        pack_kernel<T, I, 16><<<blocks, 256, 0, s>>>(
            (const I *)idx, (const T *)vals, P, off, t->P, t->N, nullptr, dm(0), dm(1), dm(2),
            dm(3), dm(4), dm(5), t->rec.as<uint8_t>(), t->keys.as<uint32_t>(), flag, partial);
    else
        pack_kernel<T, I, 32><<<blocks, 256, 0, s>>>(
            (const I *)idx, (const T *)vals, P, off, t->P, t->N, nullptr, dm(0), dm(1), dm(2),
            dm(3), dm(4), dm(5), t->rec.as<uint8_t>(), t->keys.as<uint32_t>(), flag, partial);
}

int pack_blocks(int64_t P) {
    int blocks = dev_sms() * 8;
    const int64_t need = (P + 255) / 256;
    if (need < blocks) blocks = (int)need;
    return blocks < 1 ? 1 : blocks;
}

// Pack nonzeros [off, off + P) from device buffers idx/vals (chunk-relative);
// the block partials of sum x^2 go to partial[0 .. pack_blocks(P)).
sptk_status launch_pack_chunk(sptk_tensor t, const void *idx, sptk_idx_type itype,
                              const void *vals, int64_t P, int64_t off, int *d_flag,
                              double *partial, cudaStream_t s) {
    const int blocks = pack_blocks(P);
    if (t->dtype == SPTK_F64) {
        if (itype == SPTK_IDX_I64)
            pack_dispatch<double, int64_t>(t, idx, vals, P, off, d_flag, partial, blocks, s);
        else
            pack_dispatch<double, uint32_t>(t, idx, vals, P, off, d_flag, partial, blocks, s);
    } else {
        if (itype == SPTK_IDX_I64)
            pack_dispatch<float, int64_t>(t, idx, vals, P, off, d_flag, partial, blocks, s);
        else
            pack_dispatch<float, uint32_t>(t, idx, vals, P, off, d_flag, partial, blocks, s);
    }
    count_launch();
    SPTK_CUDA(cudaGetLastError());
    return SPTK_OK;
}

sptk_status launch_pack(sptk_tensor t, const void *idx, sptk_idx_type itype, const void *vals,
                        int *d_flag, double *d_normsq, cudaStream_t s) {
    const int blocks = pack_blocks(t->P);
    DevBuf &part = t->als.partial;
    SPTK_TRY(part.reserve(sizeof(double) * blocks));
    SPTK_TRY(launch_pack_chunk(t, idx, itype, vals, t->P, 0, d_flag, part.as<double>(), s));
    return launch_sum_f64(part.as<double>(), blocks, d_normsq, s);
}

}  // namespace sptk
