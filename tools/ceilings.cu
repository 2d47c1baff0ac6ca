// ceilings.cu -- measured B200 ceilings for the MTTKRP hot path (SURVEY §8(d)
// "the B200 parameters to measure in the same run", items 1-5):
//
//   hbm_read        streaming read of a 4 GB buffer (256-bit loads)
//   gather_<loc>_<B>  random B-byte row gathers, row ids PRECOMPUTED (a streamed
//                   uint32 index array, like the MTTKRP's compact records), from
//                   a table resident in L1 (96 KB), L2 (6.4 MB), ~L2 (96 MB) or
//                   HBM (2.2 GB); lanes across the row (B/32 lanes x 32 B), 8
//                   rows in flight per lane group.  "l1" variants allocate in L1,
//                   "nol1" use L1::no_allocate (L2 -> SM path only).
//   dfma / ffma     fp64 / fp32 FMA throughput (independent chains)
//   red_f64_spread  red.global.add.f64 to distinct addresses (atomic unit rate)
//   red_f64_hot     red.global.add.f64 to one 128-byte row (contention: a hot
//                   output row of a power-law mode)
//
// Every number is useful bytes (or flops / ops) / best-of-5 CUDA-event time.
// Output: one JSON object on stdout (bench.py reads profiles/ceilings.json).
//   tma_gather4_<loc>  the same random 128-byte rows fetched by TMA
//                   (cp.async.bulk.tensor.2d ... tile::gather4: 4 rows per
//                   instruction, one issuing lane per warp, S-stage smem ring
//                   with mbarriers) -- the LSU-free gather path
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o tools/ceilings tools/ceilings.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <random>
#include <string>
#include <vector>

#define CK(x)                                                                                \
    do {                                                                                     \
        cudaError_t e_ = (x);                                                                \
        if (e_ != cudaSuccess) {                                                             \
            fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
            return 1;                                                                        \
        }                                                                                    \
    } while (0)

__device__ __forceinline__ void ld32(const double *p, double (&r)[4], bool l1) {
    if (l1)
        asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
                     : "=d"(r[0]), "=d"(r[1]), "=d"(r[2]), "=d"(r[3]) : "l"(p));
    else
        asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
                     : "=d"(r[0]), "=d"(r[1]), "=d"(r[2]), "=d"(r[3]) : "l"(p));
}

__global__ void __launch_bounds__(256) hbm_read(const double *a, int64_t n4, double *out) {
    double acc = 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += 4 * stride) {
        double r[4][4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t k = i + u * stride;
            if (k < n4) ld32(a + 4 * k, r[u], false);
            else r[u][0] = r[u][1] = r[u][2] = r[u][3] = 0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) acc += r[u][0] + r[u][1] + r[u][2] + r[u][3];
    }
    if (acc == 1.2345) out[0] = acc;
}

// G lanes per row (G = ROWB / 32), each lane 32 bytes; U rows per group in flight
template <int G, bool L1>
__global__ void __launch_bounds__(256) gather_rows(const uint32_t *__restrict__ idx, int64_t n,
                                                   const double *__restrict__ A, double *out) {
    constexpr int U = 8;
    constexpr int ROWD = G * 4;  // doubles per row
    const int q = threadIdx.x % G;
    const int64_t g0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / G;
    const int64_t gs = ((int64_t)gridDim.x * blockDim.x) / G;
    double acc = 0;
    for (int64_t k = g0; k < n; k += gs * U) {
        uint32_t row[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t kk = k + u * gs;
            uint32_t v = 0;
            if (kk < n)
                asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(idx + kk));
            row[u] = v;
        }
        double f[U][4];
#pragma unroll
        for (int u = 0; u < U; ++u) ld32(A + (int64_t)row[u] * ROWD + q * 4, f[u], L1);
#pragma unroll
        for (int u = 0; u < U; ++u) acc += (f[u][0] + f[u][1]) + (f[u][2] + f[u][3]);
    }
    if (acc == 1.2345) out[0] = acc;
}

// The slice MTTKRP's data movement without its arithmetic: per element a
// 16-byte record {row of A (uint32), row of B (uint32), value (f64)} streamed
// with L1::no_allocate, one 128-byte row of A from an L1-sized table
// (L1-allocating: the secondary factor's window) and one of B from an
// L2-resident table (L1::no_allocate: the other factor); 4 lanes x 32 B per
// row, U elements in flight per group.  An upper bound for the kernel: its
// window rows hit L1 only ~35 % of the time (ncu), here always.
template <int G>  // lanes per row: 4 = 128-byte rows (f64 R=16), 2 = 64-byte rows (f32 R=16)
__global__ void __launch_bounds__(256) pair_gather(const uint4 *__restrict__ rec, int64_t n,
                                                   const double *__restrict__ A,
                                                   const double *__restrict__ B, double *out) {
    constexpr int U = 4;
    const int q = threadIdx.x % G;
    const int64_t g0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / G;
    const int64_t gs = ((int64_t)gridDim.x * blockDim.x) / G;
    double acc = 0;
    for (int64_t k = g0; k < n; k += gs * U) {
        uint32_t ra[U], rb[U];
        double x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t kk = k + u * gs;
            uint32_t w0 = 0, w1 = 0, w2 = 0, w3 = 0;
            if (kk < n)
                asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                             : "=r"(w0), "=r"(w1), "=r"(w2), "=r"(w3) : "l"(rec + kk));
            ra[u] = w0;
            rb[u] = w1;
            x[u] = __hiloint2double((int)w3, (int)w2);
        }
        double fa[U][4], fb[U][4];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            ld32(A + (int64_t)ra[u] * (4 * G) + q * 4, fa[u], true);
            ld32(B + (int64_t)rb[u] * (4 * G) + q * 4, fb[u], false);
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v) acc += x[u] * fa[u][v] * fb[u][v];
    }
    if (acc == 1.2345) out[0] = acc;
}

// TMA gather4: lane 0 of each warp keeps S gather4 copies (4 rows each) in
// flight into a per-warp smem ring; the warp reads one word of every landed
// row set (checksum) before re-arming the slot
template <int S>
__global__ void __launch_bounds__(256) tma_gather4(const __grid_constant__ CUtensorMap tm,
                                                   const uint32_t *__restrict__ idx, int64_t n,
                                                   double *out) {
    constexpr int kRowB = 128, kSet = 4 * kRowB;
    extern __shared__ __align__(1024) uint8_t sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    uint8_t *ring = sm + (size_t)warp * S * kSet;
    uint64_t *bar = reinterpret_cast<uint64_t *>(sm + (size_t)nw * S * kSet) + warp * S;
    if (lane == 0)
        for (int k = 0; k < S; ++k)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar + k)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    const int64_t gw = (blockIdx.x * (int64_t)nw + warp), tw = (int64_t)gridDim.x * nw;
    const int64_t sets = n / 4;
    double acc = 0;
    int64_t it = 0;
    for (int64_t q = gw; q < sets; q += tw, ++it) {
        const int slot = (int)(it % S);
        const uint32_t b = (uint32_t)__cvta_generic_to_shared(bar + slot);
        if (it >= S) {  // wait for the set issued S iterations ago, consume it
            const uint32_t par = (uint32_t)((it / S - 1) & 1);
            asm volatile("{\n\t.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W;\n\t}" ::"r"(b), "r"(par) : "memory");
            acc += reinterpret_cast<const double *>(ring + slot * kSet)[lane * 2];
            __syncwarp();
        }
        if (lane == 0) {
            const uint4 r = *reinterpret_cast<const uint4 *>(idx + 4 * q);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(kSet) : "memory");
            asm volatile("cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
                         " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                         ::"r"((uint32_t)__cvta_generic_to_shared(ring + slot * kSet)), "l"(&tm), "r"(0),
                           "r"(r.x), "r"(r.y), "r"(r.z), "r"(r.w), "r"(b) : "memory");
        }
        __syncwarp();
    }
    for (int64_t k = (it > S ? it - S : 0); k < it; ++k) {  // drain
        const int slot = (int)(k % S);
        const uint32_t b = (uint32_t)__cvta_generic_to_shared(bar + slot);
        const uint32_t par = (uint32_t)((k / S) & 1);
        asm volatile("{\n\t.reg .pred p;\nW2: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W2;\n\t}" ::"r"(b), "r"(par) : "memory");
        acc += reinterpret_cast<const double *>(ring + slot * kSet)[lane * 2];
    }
    if (acc == 1.2345) out[0] = acc;
}

template <typename T>
__global__ void __launch_bounds__(256) fma_chain(T *out, int iters, T a, T b) {
    T x[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = (T)(threadIdx.x + j);
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = fma(x[j], a, b);
    T s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += x[j];
    if (s == (T)1.2345) out[0] = s;
}

__global__ void __launch_bounds__(256) red_spread(double *dst, int64_t ndst, int per_thread) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    for (int i = 0; i < per_thread; ++i) {
        const int64_t k = (t * 2654435761ull + i * 40503ull) % ndst;
        asm volatile("red.global.add.f64 [%0], %1;" ::"l"(dst + k), "d"(1.0) : "memory");
    }
}

__global__ void __launch_bounds__(256) red_hot(double *dst, int per_thread) {
    // 16 consecutive doubles = one 128-byte output row (f64 R = 16); lane -> column
    for (int i = 0; i < per_thread; ++i)
        asm volatile("red.global.add.f64 [%0], %1;" ::"l"(dst + (threadIdx.x & 15)), "d"(1.0) : "memory");
}

int main(int argc, char **argv) {
    int sms = 0, dev = 0, clk = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
    cudaEvent_t ea, eb;
    cudaEventCreate(&ea);
    cudaEventCreate(&eb);
    double *out;
    CK(cudaMalloc(&out, 64));
    auto best_ms = [&](auto launch) {
        launch();
        cudaDeviceSynchronize();
        float best = 1e30f;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(ea);
            launch();
            cudaEventRecord(eb);
            cudaEventSynchronize(eb);
            float ms;
            cudaEventElapsedTime(&ms, ea, eb);
            if (ms < best) best = ms;
        }
        return (double)best;
    };
    std::vector<std::string> items;
    auto emit = [&](const char *key, double value, const char *unit, const char *what) {
        char buf[512];
        snprintf(buf, sizeof buf, "\"%s\": {\"value\": %.1f, \"unit\": \"%s\", \"what\": \"%s\"}",
                 key, value, unit, what);
        items.push_back(buf);
        fprintf(stderr, "%-28s %12.1f %-8s %s\n", key, value, unit, what);
    };

    // ---- HBM streaming read
    const int64_t hb = (int64_t)4 << 30;
    double *H;
    CK(cudaMalloc(&H, hb));
    CK(cudaMemset(H, 0, hb));
    {
        const double ms = best_ms([&] { hbm_read<<<sms * 8, 256>>>(H, hb / 32, out); });
        emit("hbm_read", hb / ms / 1e6, "GB/s", "stream read of 4 GB, 256-bit loads");
    }
    // ---- random row gathers, precomputed ids
    const int64_t n = (int64_t)1 << 27;  // 134M gathers (uint32 ids: 512 MB streamed)
    uint32_t *idx;
    CK(cudaMalloc(&idx, n * 4));
    std::vector<uint32_t> h(n);
    struct Table { const char *loc; int64_t bytes; };
    const Table tables[] = {{"l1", 96 << 10}, {"l2", (int64_t)6400 << 10},
                            {"nearl2", (int64_t)96 << 20}, {"hbm", (int64_t)2200 << 20}};
    const int rowbs[] = {64, 128, 256, 512};
    std::mt19937_64 rng(1809);
    std::vector<uint32_t> raw(n);
    for (int64_t k = 0; k < n; ++k) raw[k] = (uint32_t)(rng() >> 32);
    for (const Table &tb : tables) {
        for (int rb : rowbs) {
            const int64_t rows = tb.bytes / rb;
            for (int64_t k = 0; k < n; ++k) h[k] = (uint32_t)(raw[k] % (uint64_t)rows);
            CK(cudaMemcpy(idx, h.data(), n * 4, cudaMemcpyHostToDevice));
            for (int l1 = 1; l1 >= 0; --l1) {
                if (tb.loc[1] == '1' && !l1) continue;  // an L1 table without L1 is the L2 case
                const unsigned grid = sms * 8;
                double ms = 0;
                auto run = [&](auto kern) { ms = best_ms([&] { kern<<<grid, 256>>>(idx, n, H, out); }); };
                switch (rb) {
                case 64: l1 ? run(gather_rows<2, true>) : run(gather_rows<2, false>); break;
                case 128: l1 ? run(gather_rows<4, true>) : run(gather_rows<4, false>); break;
                case 256: l1 ? run(gather_rows<8, true>) : run(gather_rows<8, false>); break;
                default: l1 ? run(gather_rows<16, true>) : run(gather_rows<16, false>); break;
                }
                char key[64], what[160];
                snprintf(key, sizeof key, "gather_%s_%s_%d", tb.loc, l1 ? "l1" : "nol1", rb);
                snprintf(what, sizeof what, "random %d B rows from a %.1f MB table, %s, ids streamed",
                         rb, tb.bytes / 1048576.0, l1 ? "L1-allocating" : "L1::no_allocate");
                emit(key, (double)n * rb / ms / 1e6, "GB/s", what);
            }
        }
    }
    // ---- the slice MTTKRP's access mix (record stream + L1 row + L2 row)
    {
        const int64_t np = (int64_t)1 << 26;  // 67M elements, 1 GB of records
        uint4 *rec;
        CK(cudaMalloc(&rec, np * 16));
        std::vector<uint4> hr(np);
        const int64_t rowsA = (96 << 10) / 128, rowsB = ((int64_t)6400 << 10) / 128;
        for (int64_t k = 0; k < np; ++k) {
            const uint64_t r = rng();
            hr[k] = make_uint4((uint32_t)((r >> 40) % rowsA), (uint32_t)((r & 0xffffffffu) % rowsB), 0u,
                               0x3ff00000u);  // value 1.0
        }
        CK(cudaMemcpy(rec, hr.data(), np * 16, cudaMemcpyHostToDevice));
        const double *TA = H, *TB = H + (int64_t)(1 << 20);  // disjoint tables in the 4 GB buffer
        for (int bps : {2, 3, 4}) {
            const double ms = best_ms([&] { pair_gather<4><<<sms * bps * 4, 256>>>(rec, np, TA, TB, out); });
            char key[64], what[200];
            snprintf(key, sizeof key, "pair_gather_l1_l2_128_x%d", bps);
            snprintf(what, sizeof what, "slice-MTTKRP mix: 16 B record + 128 B row from 96 KB (L1) + 128 B "
                     "row from 6.4 MB (L2, no L1); gathered row bytes / time, grid %d x SMs", bps * 4);
            emit(key, (double)np * 256 / ms / 1e6, "GB/s", what);
        }
        // 64-byte rows (fp32 R = 16): the same tables hold twice the rows; ids stay in range
        for (int bps : {2, 3, 4}) {
            const double ms = best_ms([&] { pair_gather<2><<<sms * bps * 4, 256>>>(rec, np, TA, TB, out); });
            char key[64], what[200];
            snprintf(key, sizeof key, "pair_gather_l1_l2_64_x%d", bps);
            snprintf(what, sizeof what, "slice-MTTKRP mix, 64 B rows: 16 B record + 64 B row from 48 KB (L1) + "
                     "64 B row from 3.2 MB (L2, no L1); gathered row bytes / time, grid %d x SMs", bps * 4);
            emit(key, (double)np * 128 / ms / 1e6, "GB/s", what);
        }
        cudaFree(rec);
    }
    // ---- TMA gather4 of 128-byte rows (precomputed ids, as above)
    {
        const struct { const char *loc; int64_t bytes; } tt[] = {{"l2", (int64_t)6400 << 10},
                                                               {"hbm", (int64_t)2200 << 20}};
        for (auto &tb : tt) {
            const int64_t rows = tb.bytes / 128;
            for (int64_t k = 0; k < n; ++k) h[k] = (uint32_t)(raw[k] % (uint64_t)rows);
            CK(cudaMemcpy(idx, h.data(), n * 4, cudaMemcpyHostToDevice));
            CUtensorMap tm;
            cuuint64_t gdim[2] = {16, (cuuint64_t)rows};
            cuuint64_t gstr[1] = {128};
            cuuint32_t box[2] = {16, 1}, es[2] = {1, 1};
            CUresult r = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, H, gdim, gstr,
                                                box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                                CU_TENSOR_MAP_SWIZZLE_NONE,
                                                CU_TENSOR_MAP_L2_PROMOTION_NONE,
                                                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r != CUDA_SUCCESS) {
                fprintf(stderr, "cuTensorMapEncodeTiled failed %d\n", (int)r);
                continue;
            }
            constexpr int S = 8;
            const size_t smb = 8 * (S * 512 + S * 8);
            CK(cudaFuncSetAttribute(tma_gather4<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smb));
            for (int bps : {2, 4, 6}) {
                const double ms = best_ms([&] { tma_gather4<S><<<sms * bps, 256, smb>>>(tm, idx, n, out); });
                CK(cudaGetLastError());
                char key[64], what[160];
                snprintf(key, sizeof key, "tma_gather4_%s_128_b%d", tb.loc, bps);
                snprintf(what, sizeof what, "TMA tile::gather4 of random 128 B rows from a %.1f MB table, "
                         "%d blocks/SM x 8 warps x %d sets in flight", tb.bytes / 1048576.0, bps, S);
                emit(key, (double)n * 128 / ms / 1e6, "GB/s", what);
            }
        }
    }
    // ---- FMA throughput
    {
        const int iters = 1 << 14;
        const double ms = best_ms([&] { fma_chain<double><<<sms * 16, 256>>>(out, iters, 1.0000001, 1e-9); });
        emit("dfma", 2.0 * 8 * iters * sms * 16 * 256 / ms / 1e9, "TFLOP/s", "fp64 FMA, 8 chains/thread");
        const double ms2 = best_ms([&] { fma_chain<float><<<sms * 16, 256>>>((float *)out, iters, 1.0000001f, 1e-9f); });
        emit("ffma", 2.0 * 8 * iters * sms * 16 * 256 / ms2 / 1e9, "TFLOP/s", "fp32 FMA, 8 chains/thread");
    }
    // ---- atomics
    {
        const int64_t ndst = (int64_t)1 << 24;
        double *D;
        CK(cudaMalloc(&D, ndst * 8));
        CK(cudaMemset(D, 0, ndst * 8));
        const int per = 64;
        const double ops = (double)sms * 8 * 256 * per;
        const double ms = best_ms([&] { red_spread<<<sms * 8, 256>>>(D, ndst, per); });
        emit("red_f64_spread", ops / ms / 1e6, "Gop/s", "red.global.add.f64 to random addresses in 128 MB");
        const double ms2 = best_ms([&] { red_hot<<<sms * 8, 256>>>(D, per); });
        emit("red_f64_hot", ops / ms2 / 1e6, "Gop/s", "red.global.add.f64 to one 128 B row (16 addresses)");
    }
    printf("{\"device_sms\": %d, \"sm_clock_mhz_attr\": %d", sms, clk / 1000);
    for (auto &s : items) printf(", %s", s.c_str());
    printf("}\n");
    return 0;
}
