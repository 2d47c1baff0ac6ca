// common.cuh -- shared internals of libsptk (handle, errors, launch helpers).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/sptk.h"

namespace sptk {

constexpr int kMaxModes = 6;
constexpr int kNumSMs = 148;  // B200; the runtime value is queried in dev_sms()

// ------------------------------------------------------------------ errors
void set_error(const std::string &msg);
sptk_status fail(sptk_status st, const std::string &msg);
sptk_status cuda_fail(cudaError_t e, const char *what);

#define SPTK_CUDA(expr)                                                        \
    do {                                                                       \
        cudaError_t _e = (expr);                                               \
        if (_e != cudaSuccess) return ::sptk::cuda_fail(_e, #expr);            \
    } while (0)

#define SPTK_TRY(expr)                                                         \
    do {                                                                       \
        sptk_status _s = (expr);                                               \
        if (_s != SPTK_OK) return _s;                                          \
    } while (0)

// ------------------------------------------------------------------ profile
struct Profile {
    bool on = false;
    int64_t launches = 0;         // every kernel launched by the library
    int64_t mttkrp_launches = 0;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pending;  // mttkrp spans
    double mttkrp_ms = 0.0;
};
Profile &profile();
inline void count_launch(int n = 1) { profile().launches += n; }
sptk_status mttkrp_span_begin(cudaStream_t s, cudaEvent_t *b);
sptk_status mttkrp_span_end(cudaStream_t s, cudaEvent_t b);

int dev_sms();

// ------------------------------------------------------------------ options
// Process-wide launch options (options.cu): default, else SPTK_<NAME> from the
// environment, else sptk_set_option.  Order = kOpts in options.cu.
enum Opt {
    OPT_RUN, OPT_VARIANT, OPT_SLICE, OPT_SLICE_L2_KB, OPT_SLICE_ROWS, OPT_SLICE_OTHER_FIRST,
    OPT_ROWREC, OPT_FORCE_V, OPT_GENERIC, OPT_DEBUG_DISPATCH, OPT_COPY_ORDER, OPT_DEFERRED_NORM,
    OPT_NO_GRAPH, OPT_GAMMA_INV_CHOL, OPT_USE_COPY, OPT_APPLY_TILE, OPT_APPLY_NB_MULT, OPT_TAIL_ROWS, OPT_APPLY_WAVE, OPT_APPLY_WARP,
    OPT_KEEP_KEYS, OPT_PDL, OPT_EXCHANGE, OPT_PAD_RANK, OPT_SORT_V1, OPT_PREZERO, OPT_APPLY_MMA, OPT_GJ_WARP, OPT_SIDE_PRIO, OPT_WIN, OPT_SLICE_FILL, OPT_FUSED_REDUCE, OPT_PREZERO_MB, OPT_ZERO_IN_APPLY, OPT_COUNT
};
int64_t opt(Opt o);
uint64_t options_generation();  // bumped by every sptk_set_option / sptk_reset_options
void set_dispatch(const std::string &s);  // what the last MTTKRP call ran (sptk_last_dispatch)

// ------------------------------------------------------------------ PDL
// Programmatic dependent launch: a kernel launched by launch_pdl may be
// scheduled while its stream predecessor is still finishing (its launch
// latency and block ramp-up overlap the predecessor's tail); such a kernel
// calls pdl_wait() -- griddepcontrol.wait, which returns once every
// predecessor has completed and its memory is visible -- before it reads or
// writes anything a predecessor touches.  Without the attribute the wait is a
// no-op.  Option pdl (default 1) switches the attribute off (A/B).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t s, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = opt(OPT_PDL) != 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// ------------------------------------------------------------------ memory
// RAII device buffer (cudaMallocAsync-free, plain cudaMalloc for large,
// long-lived buffers; workspaces are kept in the handle).
struct DevBuf {
    void *p = nullptr;
    size_t bytes = 0;
    DevBuf() = default;
    DevBuf(const DevBuf &) = delete;
    DevBuf &operator=(const DevBuf &) = delete;
    ~DevBuf() { release(); }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
    }
    sptk_status reserve(size_t n);  // grows (contents not kept)
    template <typename T> T *as() const { return static_cast<T *>(p); }
};

bool is_device_ptr(const void *p);

// ------------------------------------------------------------------ tensor
struct ALSWork {
    int64_t R = 0;
    DevBuf V;         // Imax x R (T)
    DevBuf V2, V3;    // further MTTKRP output buffers (pre-zeroed V, see als.cu)
    DevBuf G;         // N x R x R (f64) Gram matrices
    DevBuf L;         // R x R (f64) Cholesky factor of Gamma
    DevBuf partial;   // per-block partial sums (f64)
    DevBuf colsq;     // R (f64)
    DevBuf lam;       // R (f64)
    DevBuf scal;      // small f64 scalars (status, inner, fit ...)
    DevBuf stage;     // host<->device staging for factors
    DevBuf lamT;      // R (T) lambda in tensor dtype
    DevBuf gpart;     // per-block partial Gram matrices (f64)
    DevBuf trace;     // device fit history, one double per iteration
    DevBuf scl;       // deferred normalisation: s_m = 1/lambda_m (N x R f64), then the
                      // next MTTKRP's column scale prod_{m != n} s_m (R, tensor dtype)
    cudaStream_t side = nullptr;              // Cholesky / inverse, overlapped with MTTKRP
    cudaEvent_t ev_gram = nullptr, ev_inv = nullptr, ev_join = nullptr;
    cudaEvent_t ev_zero[8] = {};              // mode n's V buffer zeroed (side stream)
    double *hres = nullptr;                   // pinned: fit, inner, ||M||^2, ..., status
    // the instantiated iteration graph of the last sptk_cp_als call, replayed
    // by the next call when nothing it captured has changed (key: every buffer
    // address and cache key it reads, the stream, the options generation)
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    std::vector<uint64_t> graph_key;
    int64_t launches_per_iter = 0;
    void drop_graph() {
        if (exec) cudaGraphExecDestroy(exec);
        if (graph) cudaGraphDestroy(graph);
        exec = nullptr;
        graph = nullptr;
        graph_key.clear();
    }
    ~ALSWork() {
        drop_graph();
        if (hres) cudaFreeHost(hres);
        if (ev_gram) cudaEventDestroy(ev_gram);
        if (ev_inv) cudaEventDestroy(ev_inv);
        if (ev_join) cudaEventDestroy(ev_join);
        for (cudaEvent_t e : ev_zero)
            if (e) cudaEventDestroy(e);
        if (side) cudaStreamDestroy(side);
    }
};

}  // namespace sptk

struct sptk_tensor_s {
    int N = 0;
    int64_t dims[sptk::kMaxModes] = {0};
    int64_t P = 0;
    sptk_dtype dtype = SPTK_F64;
    int rec_bytes = 32;
    sptk::DevBuf rec;                           // packed records
    sptk::DevBuf perm[sptk::kMaxModes];         // uint32[P]
    sptk::DevBuf rowptr[sptk::kMaxModes];       // uint32[I_n + 1]
    bool has_perm[sptk::kMaxModes] = {false};
    sptk::DevBuf srec[sptk::kMaxModes];         // compact records in perm_n order (optional)
    bool has_srec[sptk::kMaxModes] = {false};
    bool copy_declined[sptk::kMaxModes] = {false};  // no memory for the copy: do not retry
    sptk::DevBuf wrow[sptk::kMaxModes];         // worker start rows for the copy (cached)
    int copy_sec[sptk::kMaxModes] = {-1, -1, -1, -1, -1, -1};  // copy's secondary mode
    int64_t copy_p0[sptk::kMaxModes] = {0}, copy_p1[sptk::kMaxModes] = {0};  // copy covers
                                                // permuted positions [copy_p0, copy_p1)
    int shard_n = 1, shard_r = 0;               // sptk_sptensor_set_shard
    bool copy_rowrec[sptk::kMaxModes] = {false};  // copy records carry the row index
    bool copy_win[sptk::kMaxModes] = {false};     // copy in window-major order (sort.cu)
    sptk::DevBuf soff[sptk::kMaxModes];         // slice offsets (slice kernel, cached)
    int64_t soff_key[sptk::kMaxModes][4] = {{-1, -1, -1, -1}};  // (row0, row1, nslice, S)
    int64_t row_max[sptk::kMaxModes] = {-1, -1, -1, -1, -1, -1};  // max nnz of a row (lazy)
    sptk::DevBuf rowmax_dev;                    // uint32[kMaxModes]: longest row, set by build_perm
    sptk::DevBuf sortws;                        // radix-sort workspace (cached)
    sptk::DevBuf keys;                          // uint32[N][P] sort keys emitted at ingest
                                                // (consumed by build_perm, then released)
    bool deterministic = false;                 // SPTK_CREATE_DETERMINISTIC
    sptk::DevBuf det_row, det_part;             // boundary-row partials (deterministic mode)
    int64_t wrow_key[sptk::kMaxModes][3] = {{-1, -1, -1}};  // (pos_begin, pos_end, run)
    bool perm_gather_only = false;              // SPTK_CREATE_PERM_GATHER
    std::vector<uint32_t> host_rowptr[sptk::kMaxModes];  // for partitioning (lazy)
    double normX2 = 0.0;
    // memory ledger of one build_perm call: the free device memory is queried
    // once when the call starts (the GPU is idle then) and afterwards estimated
    // from what the handle itself allocates or releases -- cudaMemGetInfo with
    // kernels in flight stalls the host for milliseconds
    bool ledger = false;
    size_t ledger_free0 = 0, ledger_total = 0, ledger_owned0 = 0;
    bool poisoned = false;
    int device = 0;
    sptk::ALSWork als;
};

namespace sptk {
constexpr int kMaxPeers = 8;  // ranks of one NVLink domain the fused exchange stores to
// Symmetric device memory (comm.cu): the same-size buffer on every rank,
// registered as an NCCL window; peer[p] is rank p's copy mapped into this
// process (NVLink load/store), mc its NVLS multicast address (one store
// reaches every rank).  Without NCCL >= 2.28 it is plain device memory.
struct SymMem {
    void *local = nullptr;
    size_t bytes = 0;
    void *win = nullptr;           // ncclWindow_t, NULL for plain device memory
    int npeer = 0;                 // ranks reachable by stores (== nranks) or 0
    char *peer[kMaxPeers] = {};
    char *mc = nullptr;
    bool nccl_mem = false;         // ncclMemAlloc'd
    int exchange = 0;              // agreed by all ranks: 0 NCCL broadcast, 1 peer stores, 2 multimem
};
}  // namespace sptk

struct sptk_comm_s {
    void *nccl = nullptr;  // ncclComm_t
    int nranks = 1;
    int rank = 0;
    bool force_sharded = false;  // SPTK_FORCE_SHARDED=1: take the N>1 code path at N=1
    sptk::SymMem sym;            // factor replicas of the sharded CP-ALS (grown on demand)
    void *devcomm = nullptr;     // ncclDevComm (multimem handle), if created
    bool devcomm_tried = false;
};

namespace sptk {
// true when the row-sharded path (partition + NCCL exchange) must be taken
inline bool sharded(const sptk_comm_s *c) { return c && (c->nranks > 1 || c->force_sharded); }
}  // namespace sptk

namespace sptk {

// record layout: value first, then nmodes uint32 indices, padded to 16/32 B
inline int record_bytes(sptk_dtype dt, int N) {
    const int vb = dt == SPTK_F64 ? 8 : 4;
    return (vb + 4 * N <= 16) ? 16 : 32;
}
inline int dtype_bytes(sptk_dtype dt) { return dt == SPTK_F64 ? 8 : 4; }
// compact permuted copy of mode n: value, then the N-1 other indices
inline int compact_bytes(sptk_dtype dt, int N) {
    const int vb = dt == SPTK_F64 ? 8 : 4;
    return (vb + 4 * (N - 1) <= 16) ? 16 : 32;
}

// --- kernels implemented in the .cu files (host launchers) ---
int pack_blocks(int64_t P);
sptk_status launch_pack_chunk(sptk_tensor t, const void *idx, sptk_idx_type itype,
                              const void *vals, int64_t P, int64_t off, int *d_flag,
                              double *partial, cudaStream_t s);
sptk_status launch_sum_f64(const double *in, int64_t n, double *out, cudaStream_t s);
sptk_status launch_pack(sptk_tensor t, const void *idx, sptk_idx_type itype, const void *vals,
                        int *d_flag, double *d_normsq, cudaStream_t s);
sptk_status build_perm_mode(sptk_tensor t, int mode, cudaStream_t s);
sptk_status ensure_sorted_copy(sptk_tensor t, int mode, cudaStream_t s);
bool build_needs_memory(sptk_tensor t, int m0, int m1);
void drop_copies(sptk_tensor t);
sptk_status merge_duplicates(sptk_tensor t, bool error_only, cudaStream_t s);
// out_zeroed: the caller already zeroed rows [row_begin, row_end) of out
// (CP-ALS zeroes the next mode's V buffer off the critical path)
sptk_status mttkrp_launch(sptk_tensor t, int mode, int64_t R, const void *const *factors,
                          const void *lambda, void *out, int64_t row_begin, int64_t row_end,
                          cudaStream_t s, bool out_zeroed = false);
sptk_status host_rowptr(sptk_tensor t, int mode, cudaStream_t s);
size_t owned_bytes(sptk_tensor t);  // device bytes held by the handle
int64_t row_max(sptk_tensor t, int mode, cudaStream_t s);  // longest row of a sorted mode
// free / total device memory: from the ledger inside build_perm, else queried
bool device_free(sptk_tensor t, size_t *free_b, size_t *total_b);
sptk_status comm_bcast_rows(sptk_comm c, void *buf, int64_t R, sptk_dtype dt,
                            const int64_t *bounds, cudaStream_t s);
sptk_status comm_allreduce_f64(sptk_comm c, double *buf, int64_t count, cudaStream_t s);
// grow c->sym to >= bytes (collective: every rank calls it with the same size)
sptk_status comm_sym_reserve(sptk_comm c, size_t bytes, cudaStream_t s);

}  // namespace sptk
