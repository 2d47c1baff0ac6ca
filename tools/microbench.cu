// microbench.cu -- B200 memory-path microbenchmarks that bound the MTTKRP
// hot path (SURVEY §8(d) "parameters to measure in the same run"):
//   1. random 32-byte record gathers from an HBM-resident array (the
//      permuted record access) -- several load flavours
//   2. sequential streaming of the same records (a mode-sorted copy)
//   3. random 128-byte row gathers from an L2-resident 6.4 MB table (factor
//      rows, NELL-2 shape) and from an HBM-resident 2 GB table (C4/C5 shape)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o tools/microbench tools/microbench.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#define CK(x)                                                                            \
    do {                                                                                 \
        cudaError_t e = (x);                                                             \
        if (e != cudaSuccess) {                                                          \
            printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);     \
            return 1;                                                                    \
        }                                                                                \
    } while (0)

__device__ __forceinline__ uint64_t mix(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

template <int V>
__device__ __forceinline__ void load32(const uint8_t *p, uint32_t (&r)[8]) {
    if constexpr (V == 0)
        asm volatile("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                       "=r"(r[6]), "=r"(r[7])
                     : "l"(p));
    else if constexpr (V == 1)
        asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                       "=r"(r[6]), "=r"(r[7])
                     : "l"(p));
    else if constexpr (V == 2) {
        asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                     : "l"(p));
        asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                     : "l"(p + 16));
    } else if constexpr (V == 3)
        asm volatile("ld.global.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                       "=r"(r[6]), "=r"(r[7])
                     : "l"(p));
    else if constexpr (V == 4)
        asm volatile("ld.global.cs.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                       "=r"(r[6]), "=r"(r[7])
                     : "l"(p));
    else {
        asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                     : "l"(p));
        r[4] = r[5] = r[6] = r[7] = 0;
    }
}

// one record per thread; idx = hash(i) mod n (random) or i (stream); U in flight
template <int V, bool RANDOM>
__global__ void __launch_bounds__(256) rec_gather(const uint8_t *rec, int64_t n, uint32_t *out) {
    constexpr int U = 4;
    uint32_t acc = 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i0 < n; i0 += stride * U) {
        uint32_t r[U][8];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t i = i0 + u * stride;
            if (i < n) {
                const uint64_t p = RANDOM ? mix((uint64_t)i) % (uint64_t)n : (uint64_t)i;
                load32<V>(rec + p * 32, r[u]);
            } else {
#pragma unroll
                for (int k = 0; k < 8; ++k) r[u][k] = 0;
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc ^= r[u][0] ^ r[u][3] ^ r[u][7];
    }
    if (acc == 0x12345678u) out[0] = acc;
}

// random 128 B rows: 4 lanes x 32 B per row, `rows` rows in the table
__global__ void __launch_bounds__(256) row_gather(const double *A, int64_t rows, int64_t n,
                                                  double *out) {
    constexpr int U = 4;
    const int q = threadIdx.x & 3;
    const int64_t g0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 2;
    const int64_t gs = ((int64_t)gridDim.x * blockDim.x) >> 2;
    double acc = 0.0;
    for (int64_t g = g0; g < n; g += gs * U) {
        double f[U][4];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t k = g + u * gs;
            const uint64_t row = mix((uint64_t)k) % (uint64_t)rows;
            if (k < n)
                asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
                             : "=d"(f[u][0]), "=d"(f[u][1]), "=d"(f[u][2]), "=d"(f[u][3])
                             : "l"(A + row * 16 + q * 4));
            else
                f[u][0] = f[u][1] = f[u][2] = f[u][3] = 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc += f[u][0] + f[u][1] + f[u][2] + f[u][3];
    }
    if (acc == 1.2345) out[0] = acc;
}

// MTTKRP-shaped access without the arithmetic: stream 32 B records (val,
// i0, i1, i2), gather two 128 B rows per record (4 lanes x 32 B) from
// L2-resident tables.  COOP=false: each 4-lane group walks its own
// contiguous run (as mttkrp_fast_kernel); COOP=true: the 8 groups of a warp
// take 8 consecutive records per step (one 256 B coalesced record load).
template <bool COOP, int WINDOW = 0>
__global__ void __launch_bounds__(256, 3) stream_gather(const uint8_t *rec, int64_t n,
                                                        const double *A1, const double *A2,
                                                        int64_t run, double *out) {
    const int q = threadIdx.x & 3;
    const int64_t gtid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int64_t s, e, stride;
    if (COOP) {
        const int64_t warp = gtid >> 5;
        const int g = (threadIdx.x & 31) >> 2;
        s = warp * run * 8 + g;
        e = min(warp * run * 8 + run * 8, n);
        stride = 8;
    } else {
        const int64_t grp = gtid >> 2;
        s = grp * run;
        e = min(s + run, n);
        stride = 1;
    }
    double acc[4] = {0, 0, 0, 0};
    for (int64_t i = s; i < e; i += 2 * stride) {
        uint32_t r[2][8];
        double f[2][2][4];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int64_t p = i + u * stride;
            if (p < e) load32<1>(rec + p * 32, r[u]);
            else r[u][3] = r[u][4] = 0, r[u][0] = r[u][1] = 0;
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
                         : "=d"(f[u][0][0]), "=d"(f[u][0][1]), "=d"(f[u][0][2]), "=d"(f[u][0][3])
                         : "l"(A1 + (uint64_t)(r[u][3] % 9200u) * 16 + q * 4));
            asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
                         : "=d"(f[u][1][0]), "=d"(f[u][1][1]), "=d"(f[u][1][2]), "=d"(f[u][1][3])
                         : "l"(A2 + (WINDOW ? (uint64_t)((blockIdx.x % 148) * WINDOW + r[u][4] % WINDOW)
                                            : (uint64_t)(r[u][4] % 28800u)) * 16 + q * 4));
        }
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v) acc[v] += __uint_as_float(r[u][0]) * f[u][0][v] * f[u][1][v];
    }
    if (acc[0] + acc[1] + acc[2] + acc[3] == 1.2345) out[0] = acc[0];
}

__global__ void fill_rec(uint8_t *rec, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        uint32_t *w = reinterpret_cast<uint32_t *>(rec + i * 32);
        const uint64_t h = mix((uint64_t)i);
        w[0] = 0x3f800000u;
        w[1] = 0;
        w[2] = (uint32_t)(i / 6400);
        w[3] = (uint32_t)(h & 0xffffffffu);
        w[4] = (uint32_t)(h >> 32);
    }
}

int main() {
    const int64_t n = 77000000;  // NELL-2 nonzeros
    uint8_t *rec;
    uint32_t *out;
    CK(cudaMalloc(&rec, n * 32));
    CK(cudaMalloc(&out, 64));
    CK(cudaMemset(rec, 1, n * 32));
    const int64_t big_rows = 17000000;  // Delicious 17M-row mode, 128 B rows (2.2 GB)
    double *A;
    CK(cudaMalloc(&A, big_rows * 128));
    CK(cudaMemset(A, 0, big_rows * 128));
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int grid = sms * 8;
    auto time_it = [&](auto launch, const char *name, double useful_bytes) {
        launch();
        cudaDeviceSynchronize();
        float best = 1e9f;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(a);
            launch();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (ms < best) best = ms;
        }
        printf("%-58s %8.3f ms  %9.1f GB/s useful\n", name, best, useful_bytes / best / 1e6);
    };
    const double rb = (double)n * 32;
    time_it([&] { rec_gather<0, true><<<grid, 256>>>(rec, n, out); }, "rec32 random  ld.nc.v8 (LDG.256)", rb);
    time_it([&] { rec_gather<1, true><<<grid, 256>>>(rec, n, out); }, "rec32 random  ld.nc.L1::no_allocate.v8", rb);
    time_it([&] { rec_gather<2, true><<<grid, 256>>>(rec, n, out); }, "rec32 random  2x ld.nc.v4 (LDG.128)", rb);
    time_it([&] { rec_gather<3, true><<<grid, 256>>>(rec, n, out); }, "rec32 random  ld.global.v8 (coherent)", rb);
    time_it([&] { rec_gather<4, true><<<grid, 256>>>(rec, n, out); }, "rec32 random  ld.global.cs.v8 (evict-first)", rb);
    time_it([&] { rec_gather<5, true><<<grid, 256>>>(rec, n, out); }, "rec16 random  ld.nc.v4 (half record)", rb / 2);
    time_it([&] { rec_gather<0, false><<<grid, 256>>>(rec, n, out); }, "rec32 stream  ld.nc.v8", rb);
    fill_rec<<<sms * 8, 256>>>(rec, n);
    CK(cudaDeviceSynchronize());
    double *T1, *T2;
    CK(cudaMalloc(&T1, 9200 * 128));
    CK(cudaMalloc(&T2, 28800 * 128));
    CK(cudaMemset(T1, 0, 9200 * 128));
    CK(cudaMemset(T2, 0, 28800 * 128));
    const double mb = (double)n * (32 + 256);
    for (int64_t run : {64, 256}) {
        const int64_t groups = (n + run - 1) / run;
        char name[128];
        snprintf(name, sizeof name, "mttkrp-shaped: per-group runs (run=%ld)", (long)run);
        time_it([&] { stream_gather<false><<<(unsigned)((groups * 4 + 255) / 256), 256>>>(rec, n, T1, T2, run, (double *)out); }, name, mb);
        const int64_t warps = (n + run * 8 - 1) / (run * 8);
        snprintf(name, sizeof name, "mttkrp-shaped: warp-cooperative (run=%ld/group)", (long)run);
        time_it([&] { stream_gather<true><<<(unsigned)((warps * 32 + 255) / 256), 256>>>(rec, n, T1, T2, run, (double *)out); }, name, mb);
        snprintf(name, sizeof name, "  ... A2 rows from a 195-row window per block (run=%ld)", (long)run);
        time_it([&] { stream_gather<true, 195><<<(unsigned)((warps * 32 + 255) / 256), 256>>>(rec, n, T1, T2, run, (double *)out); }, name, mb);
        snprintf(name, sizeof name, "  ... A2 rows from a 32-row window per block (run=%ld)", (long)run);
        time_it([&] { stream_gather<true, 32><<<(unsigned)((warps * 32 + 255) / 256), 256>>>(rec, n, T1, T2, run, (double *)out); }, name, mb);
    }
    const int64_t ng = 154000000;  // 77M nnz x 2 gathered rows
    const double gb = (double)ng * 128;
    time_it([&] { row_gather<<<grid, 256>>>(A, 50000, ng, (double *)out); }, "row128 random from 6.4 MB (L2-resident)", gb);
    time_it([&] { row_gather<<<grid, 256>>>(A, 1000000, ng, (double *)out); }, "row128 random from 128 MB (~L2 size)", gb);
    time_it([&] { row_gather<<<grid, 256>>>(A, big_rows, ng, (double *)out); }, "row128 random from 2.2 GB (HBM)", gb);
    return 0;
}
