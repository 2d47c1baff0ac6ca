// gen.cu -- device implementation of the synthetic-input generator text in
// synth/__init__.py.  NOT part of the product library: a
// separate shared object (libsynth.so) that writes inputs for large configs
// straight into device memory.  Holds none of the method's arithmetic.
// Non-fused __dmul_rn/__dadd_rn keep the power-law polynomial bit-identical
// to the numpy host version (tests/test_synth.py).
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ uint64_t draw(uint64_t seed, uint64_t stream, uint64_t i) {
    return splitmix64(seed ^ (i * 0x9E3779B97F4A7C15ull) ^ (stream * 0xD1B54A32D192ED03ull));
}

__device__ __forceinline__ double unit(uint64_t d) { return (double)(d >> 11) * 0x1.0p-53; }

struct PowCoeffs {
    double c[17];
};

__global__ void coords_kernel(uint64_t seed, int mode, int nmodes, uint32_t I, uint64_t i0,
                              int64_t count, int dist, double L, uint64_t a, uint64_t b,
                              PowCoeffs pc, uint32_t *__restrict__ out) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < count;
         k += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t d = draw(seed, (uint64_t)mode, i0 + (uint64_t)k);
        uint32_t l;
        if (dist == 0) {
            l = (uint32_t)(((d >> 32) * (uint64_t)I) >> 32);
        } else {
            const double t = __dmul_rn(unit(d), L);
            const double e = floor(t);
            const double f = __dadd_rn(t, -e);
            double y = pc.c[16];
#pragma unroll
            for (int j = 15; j >= 0; --j) y = __dadd_rn(__dmul_rn(y, f), pc.c[j]);
            y = ldexp(y, (int)e);
            int64_t r = (int64_t)floor(y) - 1;
            if (r < 0) r = 0;
            if (r > (int64_t)I - 1) r = (int64_t)I - 1;
            l = (uint32_t)((a * (uint64_t)r + b) % (uint64_t)I);
        }
        out[(size_t)k * nmodes + mode] = l;
    }
}

// same draws at arbitrary counters ids[k] (instead of i0 + k), out[k]
__global__ void coords_at_kernel(uint64_t seed, int mode, uint32_t I, const uint32_t *__restrict__ ids,
                                 int64_t count, int dist, double L, uint64_t a, uint64_t b,
                                 PowCoeffs pc, uint32_t *__restrict__ out) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < count;
         k += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t d = draw(seed, (uint64_t)mode, (uint64_t)ids[k]);
        uint32_t l;
        if (dist == 0) {
            l = (uint32_t)(((d >> 32) * (uint64_t)I) >> 32);
        } else {
            const double t = __dmul_rn(unit(d), L);
            const double e = floor(t);
            const double f = __dadd_rn(t, -e);
            double y = pc.c[16];
#pragma unroll
            for (int j = 15; j >= 0; --j) y = __dadd_rn(__dmul_rn(y, f), pc.c[j]);
            y = ldexp(y, (int)e);
            int64_t r = (int64_t)floor(y) - 1;
            if (r < 0) r = 0;
            if (r > (int64_t)I - 1) r = (int64_t)I - 1;
            l = (uint32_t)((a * (uint64_t)r + b) % (uint64_t)I);
        }
        out[k] = l;
    }
}

__global__ void values_at_kernel(uint64_t seed, int nmodes, const uint32_t *__restrict__ ids,
                                 int64_t count, double *__restrict__ out) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < count;
         k += (int64_t)gridDim.x * blockDim.x)
        out[k] = 1.0 - unit(draw(seed, (uint64_t)nmodes, (uint64_t)ids[k]));
}

__global__ void values_kernel(uint64_t seed, int nmodes, uint64_t i0, int64_t count, int f32,
                              void *__restrict__ out) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < count;
         k += (int64_t)gridDim.x * blockDim.x) {
        const double x = 1.0 - unit(draw(seed, (uint64_t)nmodes, i0 + (uint64_t)k));
        if (f32) static_cast<float *>(out)[k] = __double2float_rn(x);
        else static_cast<double *>(out)[k] = x;
    }
}

__global__ void factor_kernel(uint64_t seed, uint64_t stream, int64_t n, int f32,
                              void *__restrict__ out) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
         k += (int64_t)gridDim.x * blockDim.x) {
        const double u = unit(draw(seed, stream, (uint64_t)k));
        if (f32) static_cast<float *>(out)[k] = __double2float_rn(u);
        else static_cast<double *>(out)[k] = u;
    }
}

int grid(int64_t n) {
    int64_t b = (n + 255) / 256;
    return (int)(b > 148 * 32 ? 148 * 32 : (b < 1 ? 1 : b));
}

}  // namespace

extern "C" {

// Mode-`mode` coordinates of nonzeros i0..i0+count-1 into out[k*nmodes + mode]
// (uint32, row-major count x nmodes).  dist 0 = uniform, 1 = power-law with
// host-computed (L, a, b) and Taylor coefficients coeffs[17].
int synth_coords(uint64_t seed, int mode, int nmodes, uint32_t I, uint64_t i0, int64_t count,
                 int dist, double L, uint64_t a, uint64_t b, const double *coeffs,
                 uint32_t *out, void *stream) {
    PowCoeffs pc;
    for (int j = 0; j < 17; ++j) pc.c[j] = coeffs ? coeffs[j] : 0.0;
    coords_kernel<<<grid(count), 256, 0, (cudaStream_t)stream>>>(seed, mode, nmodes, I, i0, count,
                                                                dist, L, a, b, pc, out);
    return (int)cudaGetLastError();
}

int synth_coords_at(uint64_t seed, int mode, uint32_t I, const uint32_t *ids, int64_t count,
                    int dist, double L, uint64_t a, uint64_t b, const double *coeffs, uint32_t *out,
                    void *stream) {
    PowCoeffs pc;
    for (int j = 0; j < 17; ++j) pc.c[j] = coeffs ? coeffs[j] : 0.0;
    coords_at_kernel<<<grid(count), 256, 0, (cudaStream_t)stream>>>(seed, mode, I, ids, count, dist,
                                                                   L, a, b, pc, out);
    return (int)cudaGetLastError();
}

// fp64 values 1 - u at counters ids[k]
int synth_values_at(uint64_t seed, int nmodes, const uint32_t *ids, int64_t count, double *out,
                    void *stream) {
    values_at_kernel<<<grid(count), 256, 0, (cudaStream_t)stream>>>(seed, nmodes, ids, count, out);
    return (int)cudaGetLastError();
}

int synth_values(uint64_t seed, int nmodes, uint64_t i0, int64_t count, int f32, void *out,
                 void *stream) {
    values_kernel<<<grid(count), 256, 0, (cudaStream_t)stream>>>(seed, nmodes, i0, count, f32,
                                                                out);
    return (int)cudaGetLastError();
}

// Factor matrix A_m (I x R row-major): entry (r, c) = u(draw(seed_f, nmodes+1+m, r*R+c)).
int synth_factor(uint64_t seed_f, int nmodes, int m, int64_t I, int64_t R, int f32, void *out,
                 void *stream) {
    factor_kernel<<<grid(I * R), 256, 0, (cudaStream_t)stream>>>(
        seed_f, (uint64_t)(nmodes + 1 + m), I * R, f32, out);
    return (int)cudaGetLastError();
}

}  // extern "C"
