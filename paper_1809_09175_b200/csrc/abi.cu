// abi.cu -- C ABI entry points for tensors, perms, partitioning, profiling.
// The ABI is declared (with citations) in include/sptk.h.
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#include <algorithm>
#include <atomic>
#include <vector>
#include <mutex>
#include <thread>
#include <new>

#include "common.cuh"

namespace sptk {

static thread_local std::string g_err;

void set_error(const std::string &msg) { g_err = msg; }
sptk_status fail(sptk_status st, const std::string &msg) {
    g_err = msg;
    return st;
}
sptk_status cuda_fail(cudaError_t e, const char *what) {
    g_err = std::string("CUDA error '") + cudaGetErrorString(e) + "' in " + what;
    return SPTK_ECUDA;
}

Profile &profile() {
    static Profile p;
    return p;
}

sptk_status mttkrp_span_begin(cudaStream_t s, cudaEvent_t *b) {
    *b = nullptr;
    if (!profile().on) return SPTK_OK;
    SPTK_CUDA(cudaEventCreate(b));
    SPTK_CUDA(cudaEventRecord(*b, s));
    return SPTK_OK;
}
sptk_status mttkrp_span_end(cudaStream_t s, cudaEvent_t b) {
    if (!profile().on || !b) return SPTK_OK;
    cudaEvent_t e;
    SPTK_CUDA(cudaEventCreate(&e));
    SPTK_CUDA(cudaEventRecord(e, s));
    profile().pending.push_back({b, e});
    profile().mttkrp_launches += 1;
    return SPTK_OK;
}

// SM count per device (a process may drive several GPUs): filled once per
// device under a mutex
int dev_sms() {
    constexpr int kMaxDev = 64;
    static std::atomic<int> sms[kMaxDev];
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= kMaxDev) return kNumSMs;
    int v = sms[dev].load(std::memory_order_relaxed);
    if (v > 0) return v;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) {
        cudaGetLastError();
        v = kNumSMs;
    }
    sms[dev].store(v, std::memory_order_relaxed);
    return v;
}

sptk_status DevBuf::reserve(size_t n) {
    if (n <= bytes && p) return SPTK_OK;
    release();
    if (n == 0) return SPTK_OK;
    cudaError_t e = cudaMalloc(&p, n);
    if (e != cudaSuccess) {
        cudaGetLastError();
        p = nullptr;
        return fail(SPTK_ENOMEM, "cudaMalloc of " + std::to_string(n) + " bytes failed: " +
                                     cudaGetErrorString(e));
    }
    bytes = n;
    return SPTK_OK;
}

bool is_device_ptr(const void *p) {
    if (!p) return false;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// ------------------------------------------------------------ kernels: sum
// Deterministic fixed-order sum of `n` doubles with one block.
__global__ void sum_f64_kernel(const double *__restrict__ in, int64_t n, double *__restrict__ out) {
    __shared__ double sh[256];
    double s = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += in[i];
    sh[threadIdx.x] = s;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = sh[0];
}

sptk_status launch_sum_f64(const double *in, int64_t n, double *out, cudaStream_t s) {
    sum_f64_kernel<<<1, 256, 0, s>>>(in, n, out);
    count_launch();
    SPTK_CUDA(cudaGetLastError());
    return SPTK_OK;
}


// ------------------------------------------------------------ host ingest
// Inputs in host memory are streamed in chunks: chunk k is copied into a
// pinned staging buffer (pageable sources; several CPU threads) and DMA'd on a
// copy stream while chunk k-1 is packed on the caller's stream -- the transfer
// overlaps the pack (and its sort-key emission), device staging is two
// chunks instead of the whole COO input, and pageable arrays reach PCIe rates.
constexpr int64_t kIngestChunk = 1 << 20;  // nonzeros per chunk (SPTK_INGEST_CHUNK overrides)
static int64_t ingest_chunk() {
    static int64_t v = -1;
    if (v < 0) {
        const char *e = getenv("SPTK_INGEST_CHUNK");
        v = (e && atoll(e) >= 4096) ? (int64_t)atoll(e) : kIngestChunk;
    }
    return v;
}

static bool host_pinned(const void *p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

// two pinned staging buffers, kept for the process (pinning is slow)
struct PinnedStage {
    std::mutex mu;
    void *buf[2] = {nullptr, nullptr};
    size_t bytes = 0;
};
static PinnedStage &pinned_stage() {
    static PinnedStage p;
    return p;
}

static void parallel_copy(void *dst, const void *src, size_t n) {
    const size_t kMin = (size_t)8 << 20;
    unsigned nt = std::thread::hardware_concurrency();
    nt = std::max(1u, std::min(nt, 8u));
    if (n < kMin || nt == 1) {
        memcpy(dst, src, n);
        return;
    }
    std::vector<std::thread> th;
    const size_t per = (n + nt - 1) / nt;
    for (unsigned k = 0; k < nt; ++k) {
        const size_t a = k * per, b = std::min(n, a + per);
        if (a >= b) break;
        th.emplace_back([=] { memcpy(static_cast<char *>(dst) + a, static_cast<const char *>(src) + a, b - a); });
    }
    for (auto &x : th) x.join();
}

static sptk_status ingest_chunked(sptk_tensor t, const void *idx, sptk_idx_type itype,
                                  const void *vals, int *d_flag, double *d_norm, cudaStream_t s) {
    const int64_t P = t->P;
    const size_t irow = (itype == SPTK_IDX_I64 ? 8 : 4) * (size_t)t->N, vsz = dtype_bytes(t->dtype);
    const int64_t C = std::min<int64_t>(P, ingest_chunk());
    const int64_t nchunks = (P + C - 1) / C;
    const bool dev_i = is_device_ptr(idx), dev_v = is_device_ptr(vals);
    const bool pin_i = !dev_i && host_pinned(idx), pin_v = !dev_v && host_pinned(vals);
    const bool stage_i = !dev_i && !pin_i, stage_v = !dev_v && !pin_v;
    const size_t chunk_bytes = (size_t)C * (irow + vsz);
    DevBuf dstage, parts;
    SPTK_TRY(dstage.reserve(2 * chunk_bytes));
    const int pb = pack_blocks(C);
    SPTK_TRY(parts.reserve(sizeof(double) * (size_t)nchunks * pb));
    SPTK_CUDA(cudaMemsetAsync(parts.p, 0, sizeof(double) * (size_t)nchunks * pb, s));
    PinnedStage &ps = pinned_stage();
    std::unique_lock<std::mutex> lock(ps.mu, std::defer_lock);
    if (stage_i || stage_v) {
        lock.lock();
        if (ps.bytes < chunk_bytes) {
            for (void *&b : ps.buf)
                if (b) cudaFreeHost(b), b = nullptr;
            ps.bytes = 0;
            for (void *&b : ps.buf) SPTK_CUDA(cudaHostAlloc(&b, chunk_bytes, cudaHostAllocPortable));
            ps.bytes = chunk_bytes;
        }
    }
    cudaStream_t cs = nullptr;
    cudaEvent_t ev_copy[2] = {nullptr, nullptr}, ev_pack[2] = {nullptr, nullptr};
    sptk_status st = SPTK_OK;
    auto cleanup = [&] {
        cudaStreamSynchronize(s);
        if (cs) cudaStreamSynchronize(cs), cudaStreamDestroy(cs);
        for (int b = 0; b < 2; ++b) {
            if (ev_copy[b]) cudaEventDestroy(ev_copy[b]);
            if (ev_pack[b]) cudaEventDestroy(ev_pack[b]);
        }
    };
    if (cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) != cudaSuccess) {
        cleanup();
        return cuda_fail(cudaGetLastError(), "ingest stream");
    }
    for (int b = 0; b < 2; ++b)
        if (cudaEventCreateWithFlags(&ev_copy[b], cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&ev_pack[b], cudaEventDisableTiming) != cudaSuccess) {
            cleanup();
            return cuda_fail(cudaGetLastError(), "ingest events");
        }
    for (int64_t k = 0; k < nchunks && st == SPTK_OK; ++k) {
        const int b = (int)(k & 1);
        const int64_t off = k * C, n = std::min(C, P - off);
        char *di = dstage.as<char>() + b * chunk_bytes, *dv = di + (size_t)C * irow;
        const char *si = static_cast<const char *>(idx) + (size_t)off * irow;
        const char *sv = static_cast<const char *>(vals) + (size_t)off * vsz;
        if (k >= 2 && cudaStreamWaitEvent(cs, ev_pack[b], 0) != cudaSuccess) {  // device buffer free
            st = cuda_fail(cudaGetLastError(), "ingest wait");
            break;
        }
        if ((stage_i || stage_v) && k >= 2 && cudaEventSynchronize(ev_copy[b]) != cudaSuccess) {
            st = cuda_fail(cudaGetLastError(), "ingest wait");  // pinned buffer b free
            break;
        }
        char *hp = static_cast<char *>(ps.buf[b]);
        const void *src_i = dev_i ? (const void *)si : si, *src_v = dev_v ? (const void *)sv : sv;
        if (stage_i) {
            parallel_copy(hp, si, (size_t)n * irow);
            src_i = hp;
        }
        if (stage_v) {
            parallel_copy(hp + (size_t)C * irow, sv, (size_t)n * vsz);
            src_v = hp + (size_t)C * irow;
        }
        const void *pi = di, *pv = dv;
        if (!dev_i) {
            if (cudaMemcpyAsync(di, src_i, (size_t)n * irow, cudaMemcpyHostToDevice, cs) != cudaSuccess)
                st = cuda_fail(cudaGetLastError(), "H2D idx");
        } else {
            pi = si;
        }
        if (st == SPTK_OK && !dev_v) {
            if (cudaMemcpyAsync(dv, src_v, (size_t)n * vsz, cudaMemcpyHostToDevice, cs) != cudaSuccess)
                st = cuda_fail(cudaGetLastError(), "H2D vals");
        } else if (dev_v) {
            pv = sv;
        }
        if (st != SPTK_OK) break;
        if (cudaEventRecord(ev_copy[b], cs) != cudaSuccess ||
            cudaStreamWaitEvent(s, ev_copy[b], 0) != cudaSuccess) {
            st = cuda_fail(cudaGetLastError(), "ingest events");
            break;
        }
        st = launch_pack_chunk(t, pi, itype, pv, n, off, d_flag, parts.as<double>() + k * pb, s);
        if (st == SPTK_OK && cudaEventRecord(ev_pack[b], s) != cudaSuccess)
            st = cuda_fail(cudaGetLastError(), "ingest events");
    }
    if (st == SPTK_OK) st = launch_sum_f64(parts.as<double>(), nchunks * pb, d_norm, s);
    cleanup();  // the staging buffers are released on return
    return st;
}
}  // namespace sptk

using namespace sptk;

#define CHECK_HANDLE(t)                                                                \
    do {                                                                               \
        if (!(t)) return fail(SPTK_EINVAL, "null tensor handle");                      \
        if ((t)->poisoned) return fail(SPTK_ECUDA, "tensor handle poisoned by an earlier CUDA error"); \
    } while (0)

namespace sptk {
size_t owned_bytes(sptk_tensor t) {
    size_t b = t->rec.bytes;
    for (int m = 0; m < t->N; ++m)
        b += t->perm[m].bytes + t->rowptr[m].bytes + t->srec[m].bytes + t->wrow[m].bytes +
             t->soff[m].bytes;
    b += t->sortws.bytes + t->keys.bytes + t->det_row.bytes + t->det_part.bytes;
    const ALSWork &w = t->als;
    b += w.V.bytes + w.G.bytes + w.L.bytes + w.partial.bytes + w.colsq.bytes + w.lam.bytes +
         w.scal.bytes + w.stage.bytes + w.lamT.bytes + w.gpart.bytes + w.trace.bytes + w.scl.bytes;
    return b;
}

bool device_free(sptk_tensor t, size_t *free_b, size_t *total_b) {
    if (t->ledger) {
        const size_t owned = owned_bytes(t);
        const size_t grew = owned > t->ledger_owned0 ? owned - t->ledger_owned0 : 0;
        const size_t shrank = owned < t->ledger_owned0 ? t->ledger_owned0 - owned : 0;
        *free_b = t->ledger_free0 + shrank - std::min(t->ledger_free0 + shrank, grew);
        *total_b = t->ledger_total;
        return true;
    }
    if (cudaMemGetInfo(free_b, total_b) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return true;
}
}  // namespace sptk

extern "C" {

const char *sptk_version(void) { return "sptk 0.1 sm_100a"; }

const char *sptk_last_error(void) { return g_err.c_str(); }

sptk_status sptk_sptensor_create(int nmodes, const int64_t *dims, int64_t nnz, const void *idx,
                                 sptk_idx_type itype, const void *vals, sptk_dtype dtype,
                                 unsigned flags, void *stream, sptk_tensor *out) {
    if (!out) return fail(SPTK_EINVAL, "out is NULL");
    *out = nullptr;
    if (nmodes < 1 || nmodes > kMaxModes)
        return fail(SPTK_EUNSUPPORTED, "nmodes must be in [1, 6]");
    if (!dims) return fail(SPTK_EINVAL, "dims is NULL");
    for (int m = 0; m < nmodes; ++m)
        if (dims[m] < 1 || dims[m] >= (int64_t(1) << 32))
            return fail(SPTK_EUNSUPPORTED, "dims[m] must be in [1, 2^32)");
    if (nnz < 0) return fail(SPTK_EINVAL, "nnz < 0");
    // positions are 32-bit in the kernels with small look-ahead offsets
    if (nnz > (int64_t(1) << 32) - 4096) return fail(SPTK_EUNSUPPORTED, "nnz must be <= 2^32 - 4096");
    if (dtype != SPTK_F32 && dtype != SPTK_F64) return fail(SPTK_EINVAL, "bad dtype");
    if (itype != SPTK_IDX_I64 && itype != SPTK_IDX_U32) return fail(SPTK_EINVAL, "bad idx type");
    if (flags & ~(unsigned)(SPTK_CREATE_PERM_GATHER | SPTK_CREATE_DETERMINISTIC |
                            SPTK_CREATE_DUP_SUM | SPTK_CREATE_DUP_ERROR))
        return fail(SPTK_EUNSUPPORTED, "unknown create flag");
    if ((flags & SPTK_CREATE_DUP_SUM) && (flags & SPTK_CREATE_DUP_ERROR))
        return fail(SPTK_EINVAL, "DUP_SUM and DUP_ERROR are mutually exclusive");
    if ((flags & SPTK_CREATE_PERM_GATHER) && (flags & SPTK_CREATE_DETERMINISTIC))
        return fail(SPTK_EINVAL, "PERM_GATHER and DETERMINISTIC are mutually exclusive");
    if (nnz > 0 && (!idx || !vals)) return fail(SPTK_EINVAL, "idx/vals NULL with nnz > 0");

    cudaStream_t s = (cudaStream_t)stream;
    sptk_tensor t = new (std::nothrow) sptk_tensor_s();
    if (!t) return fail(SPTK_ENOMEM, "host allocation failed");
    t->N = nmodes;
    for (int m = 0; m < nmodes; ++m) t->dims[m] = dims[m];
    t->P = nnz;
    t->dtype = dtype;
    t->rec_bytes = record_bytes(dtype, nmodes);
    t->perm_gather_only = (flags & SPTK_CREATE_PERM_GATHER) != 0;
    t->deterministic = (flags & SPTK_CREATE_DETERMINISTIC) != 0;
    cudaGetDevice(&t->device);

    sptk_status st = SPTK_OK;
    if (nnz > 0) {
        DevBuf flag;
        const bool host_input = !is_device_ptr(idx) || !is_device_ptr(vals);
        if ((st = t->rec.reserve((size_t)t->rec_bytes * nnz)) != SPTK_OK) goto bad;
        if (!(flags & (SPTK_CREATE_DUP_SUM | SPTK_CREATE_DUP_ERROR))) {
            // emit the sort keys at ingest when they fit next to a reserve
            // (otherwise build_perm extracts them from the records per mode)
            const size_t kb = sizeof(uint32_t) * (size_t)nnz * nmodes;
            size_t free_b = 0, total_b = 0;
            if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess) {
                const size_t reserve = std::max<size_t>(total_b / 32, (size_t)4 << 30);
                if (free_b >= kb + reserve && t->keys.reserve(kb) != SPTK_OK) set_error("");
            } else {
                cudaGetLastError();
            }
        }
        if ((st = flag.reserve(16)) != SPTK_OK) goto bad;
        int *d_flag = flag.as<int>();
        double *d_norm = reinterpret_cast<double *>(flag.as<char>() + 8);
        if (cudaMemsetAsync(d_flag, 0, 8, s) != cudaSuccess) {
            st = cuda_fail(cudaGetLastError(), "memset flag");
            goto bad;
        }
        st = host_input ? ingest_chunked(t, idx, itype, vals, d_flag, d_norm, s)
                        : launch_pack(t, idx, itype, vals, d_flag, d_norm, s);
        if (st != SPTK_OK) goto bad;
        struct {
            int flag;
            int pad;
            double norm;
        } h;
        if (cudaMemcpyAsync(&h, flag.p, 16, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
            cudaStreamSynchronize(s) != cudaSuccess) {
            st = cuda_fail(cudaGetLastError(), "create: reading validation flag");
            goto bad;
        }
        if (h.flag) {
            st = fail(SPTK_ERANGE, "a coordinate is outside [0, dims[m])");
            goto bad;
        }
        t->normX2 = h.norm;
        if (flags & (SPTK_CREATE_DUP_SUM | SPTK_CREATE_DUP_ERROR)) {
            st = merge_duplicates(t, (flags & SPTK_CREATE_DUP_ERROR) != 0, s);
            if (st != SPTK_OK) goto bad;
        }
    }
    *out = t;
    return SPTK_OK;
bad:
    delete t;
    return st;
}

sptk_status sptk_sptensor_destroy(sptk_tensor t) {
    if (!t) return SPTK_OK;
    delete t;
    return SPTK_OK;
}

sptk_status sptk_sptensor_info(sptk_tensor t, int *nmodes, int64_t *dims, int64_t *nnz,
                               sptk_dtype *dtype) {
    if (!t) return fail(SPTK_EINVAL, "null tensor handle");
    if (nmodes) *nmodes = t->N;
    if (dims)
        for (int m = 0; m < t->N; ++m) dims[m] = t->dims[m];
    if (nnz) *nnz = t->P;
    if (dtype) *dtype = t->dtype;
    return SPTK_OK;
}


sptk_status sptk_sptensor_device_bytes(sptk_tensor t, int64_t *bytes) {
    if (!t || !bytes) return fail(SPTK_EINVAL, "null argument");
    *bytes = (int64_t)owned_bytes(t);
    return SPTK_OK;
}

// SPTK_DEBUG_SETUP=1: synchronise and print the host time of every build_perm phase
static double setup_clock(cudaStream_t s) {
    static int on = -1;
    if (on < 0) {
        const char *e = getenv("SPTK_DEBUG_SETUP");
        on = (e && *e && *e != '0') ? 1 : 0;
    }
    if (!on) return -1.0;
    cudaStreamSynchronize(s);
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return ts.tv_sec * 1e3 + ts.tv_nsec * 1e-6;
}

static void setup_note(const char *what, int m, double &t0, cudaStream_t s) {
    const double t1 = setup_clock(s);
    if (t1 < 0) return;
    fprintf(stderr, "[sptk] build_perm %s mode %d: %.2f ms\n", what, m, t1 - t0);
    t0 = t1;
}

sptk_status sptk_sptensor_set_shard(sptk_tensor t, int nranks, int rank) {
    CHECK_HANDLE(t);
    if (nranks < 1 || rank < 0 || rank >= nranks) return fail(SPTK_EINVAL, "bad shard");
    if (t->shard_n == nranks && t->shard_r == rank) return SPTK_OK;
    t->shard_n = nranks;
    t->shard_r = rank;
    drop_copies(t);  // rebuilt for the new row ranges by build_perm / the next MTTKRP
    return SPTK_OK;
}

sptk_status sptk_build_perm(sptk_tensor t, int mode, void *stream) {
    CHECK_HANDLE(t);
    if (mode < -1 || mode >= t->N) return fail(SPTK_EINVAL, "mode out of range");
    cudaStream_t s = (cudaStream_t)stream;
    const int m0 = mode < 0 ? 0 : mode, m1 = mode < 0 ? t->N : mode + 1;
    double tc = setup_clock(s);
    // one memory query, while the GPU is idle; the rest of the call keeps a
    // ledger.  A steady-state re-sort (perm, rowptr, sort workspace and copies
    // of the modes all present) allocates nothing and decides nothing by free
    // memory: no query at all (cudaMemGetInfo cost 1 ms of host time inside
    // the timed re-sort in some processes: 2.1 instead of 1.0 ms per mode,
    // profiles/r02/s2/bench_all_final.jsonl)
    struct LedgerScope {
        sptk_tensor t;
        ~LedgerScope() { t->ledger = false; }
    } ledger_scope{t};
    const bool needs_memory = build_needs_memory(t, m0, m1);
    if (needs_memory && cudaMemGetInfo(&t->ledger_free0, &t->ledger_total) == cudaSuccess) {
        t->ledger_owned0 = owned_bytes(t);
        t->ledger = true;
    } else if (needs_memory) {
        cudaGetLastError();
    }
    // what this call may allocate: the sort workspace, copies, (released) keys
    const void *ws0 = t->sortws.p;
    const size_t ws_bytes0 = t->sortws.bytes;
    const bool keys0 = t->keys.p != nullptr;
    int copies0 = 0;
    for (int m = 0; m < t->N; ++m) copies0 += t->has_srec[m] ? 1 : 0;
    for (int m = m0; m < m1; ++m) {  // all sorts first: their temporaries are the peak
        sptk_status st = build_perm_mode(t, m, s);
        if (st == SPTK_ECUDA) t->poisoned = true;
        if (st != SPTK_OK) return st;
        setup_note("sort", m, tc, s);
    }
    bool all = true;  // the ingest keys are consumed once every mode is sorted
    for (int m = 0; m < t->N; ++m) all = all && t->has_perm[m];
    if (all && t->keys.p && needs_memory) {
        // they also speed up the copies' secondary sorts; keep them through
        // the copies only if every copy (+ its order buffer) fits beside them
        size_t free_b = 0, total_b = 0;
        if (!device_free(t, &free_b, &total_b)) free_b = 0;
        const size_t copies = (size_t)(m1 - m0) * (compact_bytes(t->dtype, t->N) + 4) * t->P;
        if (free_b < copies + std::max<size_t>(total_b / 32, (size_t)4 << 30)) t->keys.release();
    }
    setup_note("keys check", -1, tc, s);
    for (int m = m0; m < m1; ++m) {  // then the permuted copies, while memory allows
        sptk_status st = ensure_sorted_copy(t, m, s);
        if (st == SPTK_ECUDA) t->poisoned = true;
        if (st != SPTK_OK) return st;
        setup_note("copy", m, tc, s);
    }
    // the ingest keys stay resident while they fit beside the copies (checked
    // above): a later build_perm of any mode then sorts straight from them
    // instead of re-reading the 16/32-byte records; they are a cache, released
    // first when a sort or a copy needs the memory (sort.cu).  Option
    // keep_keys = 0 releases them here (re-sorts then extract the keys).
    if (all && !opt(OPT_KEEP_KEYS)) t->keys.release();
    // keep the sort workspace for the next build_perm only while memory is
    // plentiful.  A steady-state re-sort allocates nothing, so the last
    // decision stands (the ledger replaces cudaMemGetInfo, which can stall the
    // host for tens of ms while the sort is in flight: profiles/r01/perm_timing_async.log).
    int copies1 = 0;
    for (int m = 0; m < t->N; ++m) copies1 += t->has_srec[m] ? 1 : 0;
    const bool allocated = t->sortws.p != ws0 || t->sortws.bytes != ws_bytes0 ||
                           copies1 != copies0 || keys0 != (t->keys.p != nullptr);
    size_t free_b = 0, total_b = 0;
    if (!t->sortws.p || !allocated) return SPTK_OK;
    if (device_free(t, &free_b, &total_b) && free_b < total_b / 4) t->sortws.release();
    return SPTK_OK;
}

static sptk_status copy_out(void *out, const void *src, size_t bytes, cudaStream_t s) {
    if (bytes == 0) return SPTK_OK;
    const bool dev = is_device_ptr(out);
    SPTK_CUDA(cudaMemcpyAsync(out, src, bytes,
                              dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, s));
    if (!dev) SPTK_CUDA(cudaStreamSynchronize(s));
    return SPTK_OK;
}

sptk_status sptk_get_perm(sptk_tensor t, int mode, uint32_t *out, void *stream) {
    CHECK_HANDLE(t);
    if (mode < 0 || mode >= t->N) return fail(SPTK_EINVAL, "mode out of range");
    if (!t->has_perm[mode]) return fail(SPTK_ENOPERM, "build_perm(mode) has not run");
    if (t->P > 0 && !out) return fail(SPTK_EINVAL, "out is NULL");
    return copy_out(out, t->perm[mode].p, sizeof(uint32_t) * (size_t)t->P, (cudaStream_t)stream);
}

sptk_status sptk_get_rowptr(sptk_tensor t, int mode, uint32_t *out, void *stream) {
    CHECK_HANDLE(t);
    if (mode < 0 || mode >= t->N) return fail(SPTK_EINVAL, "mode out of range");
    if (!t->has_perm[mode]) return fail(SPTK_ENOPERM, "build_perm(mode) has not run");
    if (!out) return fail(SPTK_EINVAL, "out is NULL");
    return copy_out(out, t->rowptr[mode].p, sizeof(uint32_t) * (size_t)(t->dims[mode] + 1),
                    (cudaStream_t)stream);
}

sptk_status sptk_partition_rows(const uint32_t *rowptr, int64_t In, int nranks,
                                int64_t *bounds) {
    if (!rowptr || !bounds || In < 1 || nranks < 1)
        return fail(SPTK_EINVAL, "partition_rows: bad argument");
    const uint64_t P = rowptr[In];
    bounds[0] = 0;
    bounds[nranks] = In;
    for (int g = 1; g < nranks; ++g) {
        const uint64_t target = (P * (uint64_t)g + (uint64_t)nranks - 1) / (uint64_t)nranks;
        // min r with rowptr[r] >= target (rowptr non-decreasing)
        const uint32_t *it = std::lower_bound(rowptr, rowptr + In + 1, (uint32_t)target);
        int64_t r = it - rowptr;
        if (r > In) r = In;
        if (r < bounds[g - 1]) r = bounds[g - 1];
        bounds[g] = r;
    }
    return SPTK_OK;
}

sptk_status sptk_profile_enable(int on) {
    profile().on = on != 0;
    return SPTK_OK;
}

sptk_status sptk_profile_reset(void) {
    Profile &p = profile();
    for (auto &e : p.pending) {
        cudaEventDestroy(e.first);
        cudaEventDestroy(e.second);
    }
    p.pending.clear();
    p.mttkrp_ms = 0.0;
    p.mttkrp_launches = 0;
    p.launches = 0;
    return SPTK_OK;
}

sptk_status sptk_profile_read(double *mttkrp_ms, int64_t *mttkrp_launches,
                              int64_t *kernel_launches) {
    Profile &p = profile();
    for (auto &e : p.pending) {
        float ms = 0.f;
        SPTK_CUDA(cudaEventSynchronize(e.second));
        SPTK_CUDA(cudaEventElapsedTime(&ms, e.first, e.second));
        p.mttkrp_ms += ms;
        cudaEventDestroy(e.first);
        cudaEventDestroy(e.second);
    }
    p.pending.clear();
    if (mttkrp_ms) *mttkrp_ms = p.mttkrp_ms;
    if (mttkrp_launches) *mttkrp_launches = p.mttkrp_launches;
    if (kernel_launches) *kernel_launches = p.launches;
    return SPTK_OK;
}

}  // extern "C"
