// mttkrp.cu -- host side of sptk_mttkrp: dispatch on (dtype, N, R), column
// tiles, row-range (multi-GPU) launches.  Kernels: mttkrp.cuh.
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>

#include "mttkrp.cuh"

namespace sptk {

// Nonzeros per worker (the paper's NZPTM block).  Adaptive by default
// (option "run" = 0): long runs amortise the two boundary atomics, but the
// grid must still cover every SM several times, so small tensors get short
// runs (>= 4).
static int64_t run_length(int64_t npos, int G) {
    const int64_t fixed = opt(OPT_RUN);
    if (fixed > 0) return fixed < 4 ? 4 : (fixed + 3) / 4 * 4;
    const int64_t workers_per_sm = 768 / G;  // ~3 resident 256-thread blocks
    // ~2 waves of workers (4 waves: LBNL's 868K-row mode 0.091 ms at 16
    // positions per worker vs 0.087 at 32, profiles/r02/s2/ab_tall_mode_run.log)
    const int64_t target = (int64_t)dev_sms() * workers_per_sm * 2;
    int64_t run = npos / (target > 0 ? target : 1);
    if (run > 256) run = 256;
    // short runs only where the grid would otherwise not fill the GPU (small
    // tensors: the launch is latency-bound, C1 CP-ALS -12 % at 4 vs 16)
    if (run < 4) run = 4;
    return (run + 3) / 4 * 4;
}

// -1: automatic (warp-cooperative for long rows); 0/1: forced
static int variant_setting() {
    const int64_t v = opt(OPT_VARIANT);
    return (v < -1 || v >= kNumVariants) ? -1 : (int)v;
}

template <typename T, int V>
static sptk_status launch_fast_v(int N, int G, int variant, const MttkrpArgs &a, int64_t workers,
                                 cudaStream_t s) {
    switch (N) {
    case 3: return launch_fast_tnv<T, 3, V>(G, variant, a, workers, s);
    case 4: return launch_fast_tnv<T, 4, V>(G, variant, a, workers, s);
    case 5: return launch_fast_tnv<T, 5, V>(G, variant, a, workers, s);
    default: return fail(SPTK_EINVAL, "fast MTTKRP: N must be 3..5");
    }
}

template <typename T>
static sptk_status launch_fast(int N, int V, int G, int variant, const MttkrpArgs &a,
                               int64_t workers, cudaStream_t s) {
    switch (V) {
    case 1: return launch_fast_v<T, 1>(N, G, variant, a, workers, s);
    case 2: return launch_fast_v<T, 2>(N, G, variant, a, workers, s);
    case 4: return launch_fast_v<T, 4>(N, G, variant, a, workers, s);
    case 8:
        if constexpr (sizeof(T) == 4) return launch_fast_v<T, 8>(N, G, variant, a, workers, s);
        [[fallthrough]];
    default: return fail(SPTK_EINVAL, "fast MTTKRP: bad vector width");
    }
}

static int pow2ceil(int x) {
    int g = 1;
    while (g < x) g <<= 1;
    return g;
}

static bool aligned_to(const void *p, size_t b) {
    return (reinterpret_cast<uintptr_t>(p) & (b - 1)) == 0;
}

sptk_status host_rowptr(sptk_tensor t, int mode, cudaStream_t s) {
    std::vector<uint32_t> &h = t->host_rowptr[mode];
    if (!h.empty()) return SPTK_OK;
    h.resize((size_t)t->dims[mode] + 1);
    SPTK_CUDA(cudaMemcpyAsync(h.data(), t->rowptr[mode].p, sizeof(uint32_t) * h.size(),
                              cudaMemcpyDeviceToHost, s));
    SPTK_CUDA(cudaStreamSynchronize(s));
    return SPTK_OK;
}

// Deterministic mode: sum the boundary-row partials (entries 2w, 2w+1, in
// worker order = row order) per row and store them.  One warp per segment
// head; lanes split the segment's entries (fixed assignment) and the sums are
// combined with a fixed shuffle tree, so the result does not depend on timing.
template <typename T>
__global__ void det_fixup_kernel(const uint32_t *__restrict__ drow, const T *__restrict__ dpart,
                                 int64_t nent, int R, T *__restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t k = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; k < nent; k += nw) {
        const uint32_t row = drow[k];
        if (row == kNoRow) continue;
        uint32_t prev = kNoRow;
        if (k > 0) prev = drow[k - 1];
        if (prev == kNoRow && k > 1) prev = drow[k - 2];
        if (prev == row) continue;  // not the first entry of its row
        // segment end: first valid entry with another row
        int64_t e = k + 1;
        for (;; e += 32) {
            const int64_t j = e + lane;
            const bool stop = j >= nent || (drow[j] != kNoRow && drow[j] != row);
            const uint32_t b = __ballot_sync(0xffffffffu, stop);
            if (b) {
                e += __ffs(b) - 1;
                break;
            }
        }
        for (int c0 = 0; c0 < R; c0 += 16) {
            double acc[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) acc[j] = 0.0;
            for (int64_t q = k + lane; q < e; q += 32) {
                if (drow[q] != row) continue;
                const T *p = dpart + q * R + c0;
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    if (c0 + j < R) acc[j] += (double)p[j];
            }
#pragma unroll
            for (int j = 0; j < 16; ++j) {
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) acc[j] += __shfl_xor_sync(0xffffffffu, acc[j], o);
            }
            if (lane < 16 && c0 + lane < R) {
                double v = 0.0;
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    if (j == lane) v = acc[j];
                out[(int64_t)row * R + c0 + lane] = (T)v;
            }
        }
    }
}

// out[0 .. words) = 0, 16-byte stores where aligned
__global__ void __launch_bounds__(256) zero_words_kernel(uint32_t *__restrict__ out, int64_t words) {
    pdl_wait();
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int64_t head = (int64_t)(((16 - (reinterpret_cast<uintptr_t>(out) & 15)) & 15) / 4);
    if (head > words) head = words;
    for (int64_t i = t0; i < head; i += stride) out[i] = 0u;
    uint4 *v = reinterpret_cast<uint4 *>(out + head);
    const int64_t nv = (words - head) / 4;
    for (int64_t i = t0; i < nv; i += stride) v[i] = make_uint4(0u, 0u, 0u, 0u);
    for (int64_t i = head + nv * 4 + t0; i < words; i += stride) out[i] = 0u;
}

// start row of every worker: the largest r with rowptr[r] <= s (binary search)
__global__ void worker_rows_kernel(const uint32_t *__restrict__ rowptr, int64_t In, int64_t pb,
                                   int64_t run, int64_t nworkers, uint32_t *__restrict__ wrow) {
    for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < nworkers;
         w += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = pb + w * run;
        int64_t lo = 0, hi = In - 1;  // invariant: rowptr[lo] <= s
        while (lo < hi) {
            const int64_t mid = (lo + hi + 1) >> 1;
            if ((int64_t)__ldg(rowptr + mid) <= s) lo = mid;
            else hi = mid - 1;
        }
        wrow[w] = (uint32_t)lo;
    }
}

static sptk_status worker_rows(sptk_tensor t, int mode, int64_t pb, int64_t pe, int64_t run,
                               int64_t workers, cudaStream_t s) {
    int64_t *key = t->wrow_key[mode];
    if (key[0] == pb && key[1] == pe && key[2] == run && t->wrow[mode].p) return SPTK_OK;
    SPTK_TRY(t->wrow[mode].reserve(sizeof(uint32_t) * workers));
    int64_t blocks = (workers + 255) / 256;
    if (blocks > (int64_t)dev_sms() * 16) blocks = (int64_t)dev_sms() * 16;
    worker_rows_kernel<<<(unsigned)blocks, 256, 0, s>>>(t->rowptr[mode].as<uint32_t>(),
                                                        t->dims[mode], pb, run, workers,
                                                        t->wrow[mode].as<uint32_t>());
    count_launch();
    SPTK_CUDA(cudaGetLastError());
    key[0] = pb;
    key[1] = pe;
    key[2] = run;
    return SPTK_OK;
}

// Slice traversal (mttkrp_slice_kernel): soff[(r - row0)(K + 1) + k] = first
// position of row r's segment of the copy whose secondary index is >= k*S
// (binary search: the copy is sorted by the secondary index inside a row).
__global__ void slice_offsets_kernel(const uint8_t *__restrict__ srec, int rc, int word,
                                     const uint32_t *__restrict__ rowptr, int64_t row0,
                                     int64_t rows, int K, int64_t S, uint32_t *__restrict__ soff) {
    const int64_t n = rows * (K + 1);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = row0 + i / (K + 1);
        const int k = (int)(i % (K + 1));
        uint32_t lo = __ldg(rowptr + r), hi = __ldg(rowptr + r + 1);
        if (k < K) {
            const uint64_t target = (uint64_t)k * S;
            while (lo < hi) {
                const uint32_t mid = lo + ((hi - lo) >> 1);
                const uint32_t key =
                    __ldg(reinterpret_cast<const uint32_t *>(srec + (size_t)mid * rc) + word);
                if (key < target) lo = mid + 1;
                else hi = mid;
            }
        } else {
            lo = hi;  // end of the row
        }
        soff[i] = lo;
    }
}

// Rows of A_a per slice.  Measured (profiles/r01/sweep_slice.log): 1024-4096
// rows are within ~2-3 %; fp64 is best at ~512 KB of A_a per slice (R = 16:
// 4096 rows, R = 64: 1024), fp32 at 2048 rows --
// the slices keep the block's 8 warps sweeping the same window of A_a (their
// reuse is temporal, the window need not be L1-resident), while longer slices
// mean fewer partial flushes.  One slice (no slicing) loses the alignment.
constexpr int64_t kSliceRows = 2048;          // fp32
constexpr int64_t kSliceBytesF64 = 512 << 10;  // fp64: 512 KB of A_a rows (R=16: 4096, R=64: 1024)
// When A_a itself exceeds L2 (Amazon shape), a slice is instead an L2-sized
// window of A_a: blocks are scheduled slice-major (grid.x = row blocks runs
// fastest), so the whole GPU sweeps one window at a time and the A_a gathers
// hit L2 instead of HBM.
constexpr int64_t kSliceL2Bytes = 32 << 20;
static int64_t slice_l2_bytes() {  // option slice_l2_kb (tests force the window regime)
    const int64_t kb = opt(OPT_SLICE_L2_KB);
    return kb > 0 ? kb << 10 : kSliceL2Bytes;
}

// L2 policy of the other factors' gathers in the slice kernel: in the L2-window
// regime (A_a > L2 budget) they are evicted first so the window stays
// resident (Amazon -4 %); otherwise evict_last like every factor row (LBNL:
// evict_first loses 4 %).  Option slice_other_first = 0/1 overrides.
static int slice_other_first(bool l2_window) {
    const int64_t v = opt(OPT_SLICE_OTHER_FIRST);
    return v >= 0 ? (v ? 1 : 0) : (l2_window ? 1 : 0);
}

static int64_t slice_rows(size_t es, int64_t row_bytes) {  // option slice_rows overrides
    const int64_t r = opt(OPT_SLICE_ROWS);
    if (r > 0) return r;
    if (es == 8) return std::min<int64_t>(8192, std::max<int64_t>(512, kSliceBytesF64 / row_bytes));
    return kSliceRows;
}

// Number of slices for the slice traversal of `mode` over rows [r0, r1), or
// 0 when it does not apply: the copy must be ordered by a secondary mode a
// with more than one slice of rows, rows must be long enough to leave >= 32
// nonzeros per (row, slice) and balanced (the block waits for its longest
// row), and the grid must fill the GPU.  *S = rows of A_a per slice.
static int slice_count(sptk_tensor t, int mode, int64_t r0, int64_t r1, int64_t nnz,
                       int64_t row_bytes, cudaStream_t s, int64_t *S) {
    const int a = t->copy_sec[mode];
    if (a < 0 || t->deterministic || !opt(OPT_SLICE) || r1 <= r0) return 0;
    const int64_t rows = r1 - r0;
    int64_t sa = slice_rows(dtype_bytes(t->dtype), row_bytes);
    if (t->dims[a] * row_bytes > slice_l2_bytes()) {
        sa = std::max<int64_t>(sa, slice_l2_bytes() / row_bytes);
        // L2-window regime: short rows would leave few nonzeros per (row,
        // window); widen the windows (up to 2x) to keep ~96 per run (measured
        // on Amazon's 354-nonzero rows: 32 -> 57 MB windows, -7 %)
        const int64_t k32 = (t->dims[a] + sa - 1) / sa;
        const int64_t kfit = std::max<int64_t>(2, nnz / (rows * 96));
        if (kfit < k32) sa = std::min<int64_t>(2 * sa, (t->dims[a] + kfit - 1) / kfit);
    }
    // small grids (LBNL's 1.6K-row modes: 200 row groups x 2 slices = 400
    // blocks, 2.7 per SM) fill the GPU unevenly: halve the slices' rows while
    // the grid is under slice_fill blocks per SM and runs keep >= 64 nonzeros
    // (measured: 1024-row slices -17 % on those modes, +17 % on the 4.2K-row
    // ones, profiles/r02/ab_lbnl_slice_rows.log)
    if (opt(OPT_SLICE_ROWS) <= 0 && t->dims[a] * row_bytes <= slice_l2_bytes()) {
        const int64_t fill = opt(OPT_SLICE_FILL) * (int64_t)dev_sms();
        while (sa > 512 && ((rows + 7) / 8) * ((t->dims[a] + sa - 1) / sa) < fill &&
               nnz >= 64 * ((t->dims[a] + sa / 2 - 1) / (sa / 2)) * rows)
            sa /= 2;
    }
    const int64_t K = (t->dims[a] + sa - 1) / sa;
    if (K < 2 || K > 65535) return 0;
    if (opt(OPT_SLICE) == 2) {  // forced (tests): structural conditions only
        *S = sa;
        return (int)K;
    }
    if (nnz < 32 * K * rows) return 0;
    if (((rows + 7) / 8) * K < 2 * (int64_t)dev_sms()) return 0;
    const int64_t mx = row_max(t, mode, s);
    if (mx < 0 || mx * rows > 2 * nnz) return 0;  // longest row > 2x the mean
    *S = sa;
    return (int)K;
}

static sptk_status slice_offsets(sptk_tensor t, int mode, int64_t r0, int64_t r1, int K,
                                 int64_t S, cudaStream_t s) {
    int64_t *key = t->soff_key[mode];
    if (key[0] == r0 && key[1] == r1 && key[2] == K && key[3] == S && t->soff[mode].p)
        return SPTK_OK;
    const int64_t n = (r1 - r0) * (K + 1);
    SPTK_TRY(t->soff[mode].reserve(sizeof(uint32_t) * n));
    const int a = t->copy_sec[mode];
    const int word = (int)(dtype_bytes(t->dtype) / 4) + (a < mode ? a : a - 1);
    int64_t blocks = (n + 255) / 256;
    if (blocks > (int64_t)dev_sms() * 16) blocks = (int64_t)dev_sms() * 16;
    const int rc = compact_bytes(t->dtype, t->N);
    slice_offsets_kernel<<<(unsigned)blocks, 256, 0, s>>>(
        t->srec[mode].as<uint8_t>() - (size_t)t->copy_p0[mode] * rc, rc, word,
        t->rowptr[mode].as<uint32_t>(), r0, r1 - r0, K, S, t->soff[mode].as<uint32_t>());
    count_launch();
    SPTK_CUDA(cudaGetLastError());
    key[0] = r0;
    key[1] = r1;
    key[2] = K;
    key[3] = S;
    return SPTK_OK;
}

sptk_status mttkrp_launch(sptk_tensor t, int mode, int64_t R, const void *const *factors,
                          const void *lambda, void *out, int64_t row_begin, int64_t row_end,
                          cudaStream_t s, bool out_zeroed) {
    const int64_t In = t->dims[mode];
    const size_t es = dtype_bytes(t->dtype);
    if (row_end <= row_begin) return SPTK_OK;
    if (!out_zeroed) {   // zero the output rows (a kernel, not a memset node: PDL chains through it)
        const int64_t words = (row_end - row_begin) * R * (int64_t)es / 4;
        uint32_t *o = reinterpret_cast<uint32_t *>(static_cast<char *>(out) + (size_t)row_begin * R * es);
        int64_t blocks = (words / 4 + 255) / 256;
        blocks = std::max<int64_t>(1, std::min<int64_t>(blocks, (int64_t)dev_sms() * 8));
        SPTK_CUDA(launch_pdl(zero_words_kernel, dim3((unsigned)blocks), dim3(256), 0, s, o, words));
        count_launch();
    }
    int64_t pb = 0, pe = t->P;
    if (row_begin != 0 || row_end != In) {
        SPTK_TRY(host_rowptr(t, mode, s));
        pb = t->host_rowptr[mode][row_begin];
        pe = t->host_rowptr[mode][row_end];
    }
    if (pe <= pb) return SPTK_OK;

    SPTK_TRY(ensure_sorted_copy(t, mode, s));
    // the copy serves this call if it covers the call's positions (a shard's
    // copy covers only its own row range)
    bool copy = t->has_srec[mode] && pb >= t->copy_p0[mode] && pe <= t->copy_p1[mode] &&
                opt(OPT_USE_COPY) != 0;
    // a window-major copy holds rows out of order: only whole-mode calls, on
    // the cooperative kernel reading rows from the records
    const bool win = copy && t->copy_win[mode];
    if (win && (row_begin != 0 || row_end != In)) copy = false;
    MttkrpArgs a{};
    a.rec = t->rec.as<uint8_t>();  // the paper's traversal: gather through perm_n
    a.perm = t->perm[mode].as<uint32_t>();
    a.pos_begin = pb;
    a.pos_end = pe;
    a.ld = R;
    a.mode = mode;
    a.N = t->N;
    a.rb = t->rec_bytes;
    for (int m = 0; m < t->N; ++m) a.A[m] = (m == mode) ? nullptr : factors[m];
    a.lambda = lambda;

    a.out = out;

    // Lane vector width V: the widest power of two <= 32 bytes that divides R
    // and to which every factor / out / lambda pointer is aligned (rows then
    // start on V-element boundaries).  32-byte vectors are the measured best;
    // narrower ones keep any R on the fast path.  The perm-gather layout is
    // compiled for 32-byte vectors only.
    int V = 32 / (int)es;
    auto ok_v = [&](int v) {
        const size_t b = (size_t)v * es;
        if (R % v != 0 || !aligned_to(out, b) || (lambda && !aligned_to(lambda, b))) return false;
        for (int m = 0; m < t->N; ++m)
            if (m != mode && !aligned_to(factors[m], b)) return false;
        return true;
    };
    while (V > 1 && !ok_v(V)) V >>= 1;
    const int64_t v_cap = opt(OPT_FORCE_V);  // cap the lane vector width (tests, tuning)
    if (v_cap > 0)
        while (V > 1 && V > v_cap) V >>= 1;
    bool fast = t->N >= 3 && t->N <= 5 && ok_v(V) &&
                (copy || V * (int)es == 32) && !opt(OPT_GENERIC);
    const int G0 = fast ? pow2ceil((int)((R < 32 * V ? R : 32 * V) / V)) : (R <= 16 ? 4 : 32);
    a.run = run_length(pe - pb, G0);
    // warp-cooperative steps pay off when rows are long (few boundary steps)
    const int64_t rows = row_end - row_begin;
    int var = 0;
    if (win && copy && !(fast && G0 < 32)) copy = false;  // no cooperative kernel for this R
    if (fast && copy && win) {
        var = 1;
        // ~512 positions per warp: the chunks in flight then span about one
        // window of the secondary factor (in-flight positions x 16 B of A_a)
        a.run = std::max<int64_t>(1, 512 / (32 / G0));
        a.win = 1;
    } else if (fast && copy && G0 < 32) {
        var = variant_setting();
        // measured (profiles/r01/sweep_*.log): a win for >= 4 groups per warp on
        // rows averaging >= 64 nonzeros, a loss on short rows and for 2 groups
        if (var < 0) var = ((pe - pb) >= 64 * rows && G0 <= 8) ? 1 : 0;
    }
    const int64_t chunk = var == 1 ? a.run * (32 / G0) : a.run;
    const int64_t workers = (pe - pb + chunk - 1) / chunk;
    if (t->deterministic && !(fast && copy))
        return fail(SPTK_EUNSUPPORTED,
                    "deterministic MTTKRP needs the permuted-copy fast path (N in 3..5, "
                    "element-aligned factors/out/lambda, default layout)");
    if (t->deterministic) {
        SPTK_TRY(t->det_row.reserve(sizeof(uint32_t) * 2 * workers));
        SPTK_TRY(t->det_part.reserve(es * 2 * workers * R));
        a.drow = t->det_row.as<uint32_t>();
        a.dpart = t->det_part.p;
    }
    a.rowrec = copy && t->copy_rowrec[mode] && var == 0 && opt(OPT_ROWREC) != 0;
    if (fast && copy) {  // stream the compact permuted copy instead
        if (!a.win) SPTK_TRY(worker_rows(t, mode, pb, pe, chunk, workers, s));
        // indexed by absolute position: base shifted back by the copy's first position
        a.rec = t->srec[mode].as<uint8_t>() -
                (size_t)t->copy_p0[mode] * compact_bytes(t->dtype, t->N);
        a.perm = nullptr;
        a.rowptr = t->rowptr[mode].as<uint32_t>();
        a.wrow = t->wrow[mode].as<uint32_t>();
    }

    // slice traversal: one column tile (R <= 32 V), 32-byte vectors, the copy
    int64_t S = 0;
    int K = 0;
    if (fast && copy && !a.win && R <= 32 * V)
        K = slice_count(t, mode, row_begin, row_end, pe - pb, R * (int64_t)es, s, &S);
    if (K > 0) {
        SPTK_TRY(slice_offsets(t, mode, row_begin, row_end, K, S, s));
        a.soff = t->soff[mode].as<uint32_t>();
        a.row0 = row_begin;
        a.row1 = row_end;
        a.nslice = K;
        a.sec = t->copy_sec[mode];
        a.other_first = slice_other_first(t->dims[a.sec] * R * (int64_t)es > slice_l2_bytes());
        var = 2;
    }

    {
        static const char *kind[] = {"fast", "coop", "slice"};
        std::string d = !fast ? "generic" : !copy ? "perm_gather" : kind[var];
        if (fast && copy && var == 0 && a.rowrec) d += "_rowrec";
        if (a.win) d += "_window";
        if (var == 2 && t->dims[a.sec] * R * (int64_t)es > slice_l2_bytes()) d += "_l2window";
        if (t->deterministic) d += "+det";
        d += " V" + std::to_string(fast ? V : 1);
        set_dispatch(d);
    }
    if (opt(OPT_DEBUG_DISPATCH))
        fprintf(stderr, "[sptk] mttkrp mode %d rows [%lld,%lld) R %lld: %s V %d G0 %d variant %d "
                "copy %d sec %d slices %d x %lld rows\n", mode, (long long)row_begin,
                (long long)row_end, (long long)R, fast ? "fast" : "generic", V, G0, var,
                (int)copy, t->copy_sec[mode], K, (long long)S);

    cudaEvent_t ev;
    SPTK_TRY(mttkrp_span_begin(s, &ev));
    if (fast) {
        const int64_t tile = 32 * V;
        for (int64_t c0 = 0; c0 < R; c0 += tile) {
            a.col0 = (int)c0;
            a.ncols = (int)((R - c0) < tile ? (R - c0) : tile);
            const int G = pow2ceil(a.ncols / V);
            if (t->dtype == SPTK_F64) SPTK_TRY(launch_fast<double>(t->N, V, G, var, a, workers, s));
            else SPTK_TRY(launch_fast<float>(t->N, V, G, var, a, workers, s));
        }
    } else {
        const int G = R <= 16 ? 4 : 32;
        const int64_t tile = (int64_t)G * 4;
        for (int64_t c0 = 0; c0 < R; c0 += tile) {
            a.col0 = (int)c0;
            a.ncols = (int)((R - c0) < tile ? (R - c0) : tile);
            if (t->dtype == SPTK_F64) SPTK_TRY(launch_generic<double>(G, a, workers, s));
            else SPTK_TRY(launch_generic<float>(G, a, workers, s));
        }
    }
    if (t->deterministic) {
        const int64_t nent = 2 * workers;
        int64_t blocks = (nent * 32 + 255) / 256;
        if (blocks > (int64_t)dev_sms() * 16) blocks = (int64_t)dev_sms() * 16;
        if (t->dtype == SPTK_F64)
            det_fixup_kernel<double><<<(unsigned)blocks, 256, 0, s>>>(
                a.drow, static_cast<const double *>(a.dpart), nent, (int)R, static_cast<double *>(out));
        else
            det_fixup_kernel<float><<<(unsigned)blocks, 256, 0, s>>>(
                a.drow, static_cast<const float *>(a.dpart), nent, (int)R, static_cast<float *>(out));
        count_launch();
        SPTK_CUDA(cudaGetLastError());
    }
    SPTK_TRY(mttkrp_span_end(s, ev));
    return SPTK_OK;
}

}  // namespace sptk

using namespace sptk;

extern "C" sptk_status sptk_set_tuning(int variant, int64_t run) {
    if (variant >= kNumVariants || variant < -2 || run < -2)
        return fail(SPTK_EINVAL, "set_tuning: variant in [-2, 1], run >= -2");
    if (variant >= 0) SPTK_TRY(sptk_set_option("variant", variant));
    if (variant == -2) SPTK_TRY(sptk_set_option("variant", -1));  // back to automatic
    if (run > 0) SPTK_TRY(sptk_set_option("run", run < 4 ? 4 : (run + 3) / 4 * 4));
    if (run == -2) SPTK_TRY(sptk_set_option("run", 0));  // back to adaptive
    return SPTK_OK;
}

extern "C" sptk_status sptk_mttkrp(sptk_tensor t, int mode, int64_t R,
                                   const void *const *factors, const void *lambda, void *out,
                                   sptk_comm comm, void *stream) {
    if (!t) return fail(SPTK_EINVAL, "null tensor handle");
    if (t->poisoned) return fail(SPTK_ECUDA, "tensor handle poisoned by an earlier CUDA error");
    if (mode < 0 || mode >= t->N) return fail(SPTK_EINVAL, "mode out of range");
    if (R < 1 || R > (int64_t(1) << 20)) return fail(SPTK_EINVAL, "R must be in [1, 2^20]");
    if (!factors || !out) return fail(SPTK_EINVAL, "factors/out is NULL");
    for (int m = 0; m < t->N; ++m)
        if (m != mode && !factors[m]) return fail(SPTK_EINVAL, "factors[m] is NULL");
    if (!t->has_perm[mode]) return fail(SPTK_ENOPERM, "build_perm(mode) has not run");
    cudaStream_t s = (cudaStream_t)stream;
    sptk_status st;
    if (!sharded(comm)) {
        st = mttkrp_launch(t, mode, R, factors, lambda, out, 0, t->dims[mode], s);
    } else {
        st = host_rowptr(t, mode, s);
        std::vector<int64_t> b(comm->nranks + 1);
        if (st == SPTK_OK)
            st = sptk_partition_rows(t->host_rowptr[mode].data(), t->dims[mode], comm->nranks,
                                     b.data());
        if (st == SPTK_OK)
            st = mttkrp_launch(t, mode, R, factors, lambda, out, b[comm->rank],
                               b[comm->rank + 1], s);
        if (st == SPTK_OK) st = comm_bcast_rows(comm, out, R, t->dtype, b.data(), s);
    }
    if (st == SPTK_ECUDA) t->poisoned = true;
    return st;
}

extern "C" sptk_status sptk_mttkrp_rows(sptk_tensor t, int mode, int64_t R,
                                        const void *const *factors, const void *lambda,
                                        void *out, int64_t row_begin, int64_t row_end,
                                        void *stream) {
    if (!t) return fail(SPTK_EINVAL, "null tensor handle");
    if (t->poisoned) return fail(SPTK_ECUDA, "tensor handle poisoned by an earlier CUDA error");
    if (mode < 0 || mode >= t->N) return fail(SPTK_EINVAL, "mode out of range");
    if (R < 1 || R > (int64_t(1) << 20)) return fail(SPTK_EINVAL, "R must be in [1, 2^20]");
    if (!factors || !out) return fail(SPTK_EINVAL, "factors/out is NULL");
    for (int m = 0; m < t->N; ++m)
        if (m != mode && !factors[m]) return fail(SPTK_EINVAL, "factors[m] is NULL");
    if (row_begin < 0 || row_end > t->dims[mode] || row_begin > row_end)
        return fail(SPTK_EINVAL, "row range outside [0, I_n]");
    if (!t->has_perm[mode]) return fail(SPTK_ENOPERM, "build_perm(mode) has not run");
    sptk_status st = mttkrp_launch(t, mode, R, factors, lambda, out, row_begin, row_end,
                                   (cudaStream_t)stream);
    if (st == SPTK_ECUDA) t->poisoned = true;
    return st;
}
