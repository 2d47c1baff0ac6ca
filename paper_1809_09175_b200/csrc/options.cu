// options.cu -- process-wide launch options (traversal selection and tuning).
//
// Every option starts from its default, or from the environment variable
// SPTK_<NAME> (upper case) when that is set, and can be changed at run time
// with sptk_set_option -- the tests force each MTTKRP traversal in-process
// this way, and sptk_last_dispatch() reports which traversal a call ran.
#include <stdlib.h>
#include <string.h>

#include <atomic>
#include <mutex>
#include <string>

#include "common.cuh"

namespace sptk {

namespace {
struct OptDef {
    const char *name;
    int64_t def;
};
// keep in the order of enum Opt (common.cuh)
constexpr OptDef kOpts[] = {
    {"run", 0},                 // positions per worker: 0 adaptive, > 0 fixed
    {"variant", -1},            // fast kernel worker shape: -1 auto, 0 per-group, 1 warp-coop
    {"slice", 1},               // 0 disables the slice traversal, 2 forces it wherever the
                                //   copy has a secondary mode (no profitability test)
    {"slice_l2_kb", 32768},     // L2 window of the slice traversal (KB of A_a rows)
    {"slice_rows", 0},          // rows of A_a per slice: 0 auto
    {"slice_other_first", -1},  // slice kernel: other factors evict-first (-1 auto)
    {"rowrec", 1},              // per-group kernel reads the row from the record's spare word
    {"force_v", 0},             // cap of the lane vector width (elements), 0 = none
    {"generic", 0},             // 1 forces the generic (scalar, runtime-N) kernel
    {"debug_dispatch", 0},      // one stderr line per MTTKRP launch
    {"copy_order", 1},          // copies' secondary key: 1 by balance (largest factor for
                                //   power-law modes), 2 always the shortest, 0 none
    {"deferred_norm", 1},       // CP-ALS deferred column normalisation (R <= 32)
    {"no_graph", 0},            // CP-ALS: 1 disables the CUDA-graph replay
    {"gamma_inv_chol", 0},      // CP-ALS: 1 = Cholesky inverse instead of Gauss-Jordan
    {"use_copy", 1},            // 0: MTTKRP gathers through perm_n even where a copy exists
    {"apply_tile", 64},         // CP-ALS apply_gram: rows of V per tile (tuning)
    {"apply_nb_mult", 1},       // CP-ALS apply_gram: block cap = mult x 8 x SMs (tuning)
    {"tail_rows", 8192},        // CP-ALS: modes up to this many rows finalise in apply_gram's last block
    {"apply_wave", 1},          // CP-ALS apply_gram: grid capped at one wave of resident blocks
    {"apply_warp", 1},          // CP-ALS: warp-private apply_gram kernel (0: shared-memory tiles)
    {"keep_keys", 1},           // keep the ingest sort keys resident after build_perm
    {"pdl", 1},                 // programmatic dependent launch of the MTTKRP / ALS kernels
    {"exchange", -1},           // sharded CP-ALS row exchange: -1 best available, 0 NCCL
                                //   broadcast, 1 peer stores, 2 NVLS multimem stores
    {"pad_rank", 1},            // CP-ALS: R not a multiple of the 32-byte lane vector runs on
                                //   factors padded with zero columns (0: stride R)
    {"sort_v1", 0},             // 1: round-1 radix downsweep (A/B)
    {"prezero", 1},             // CP-ALS: MTTKRP outputs of >= 256 MB zeroed on the side stream, off
                                //   the critical path (2: every output, tests)
    {"apply_mma", 1},           // CP-ALS apply_gram on the FP64 tensor cores (DMMA) for R = 8 / 16
    {"gj_warp", 1},             // CP-ALS: one-warp register Gauss-Jordan inverse for R <= 32
    {"side_prio", -1},          // CP-ALS side stream (inverse, zeroing) at the highest priority:
                                //   -1 for tensors of >= 2^20 nonzeros, 1 always, 0 never
    {"win", 0},                 // > 0: window-major copies for modes with few rows whose secondary
                                //   factor spans >= 2 x win L2 windows (power-law tensors)
    {"slice_fill", 6},          // slice traversal: halve the slices until the grid has this many
                                //   blocks per SM (0 = off)
    {"fused_reduce", 1},        // CP-ALS: a large mode's reductions + finalise (+ fit) in one launch
    {"prezero_mb", 256},        // CP-ALS (prezero 1): outputs of at least this many MB are pre-zeroed
    {"zero_in_apply", 0},       // CP-ALS: pre-zero from extra blocks of the previous mode's apply
};

static_assert(sizeof(kOpts) / sizeof(kOpts[0]) == OPT_COUNT, "kOpts must list every Opt, in order");

std::mutex g_mu;
std::atomic<bool> g_init{false};
std::atomic<int64_t> g_val[OPT_COUNT];

int64_t env_value(const char *name, int64_t def) {
    std::string env = "SPTK_";
    for (const char *c = name; *c; ++c) env += (char)(*c >= 'a' && *c <= 'z' ? *c - 32 : *c);
    const char *e = getenv(env.c_str());
    if (!e || !*e) return def;
    char *end = nullptr;
    const long long v = strtoll(e, &end, 10);
    return end == e ? def : (int64_t)v;
}

void init_locked() {
    for (int i = 0; i < OPT_COUNT; ++i) g_val[i] = env_value(kOpts[i].name, kOpts[i].def);
    // legacy spelling: SPTK_GAMMA_INV=chol
    if (const char *g = getenv("SPTK_GAMMA_INV"))
        if (g[0] == 'c') g_val[OPT_GAMMA_INV_CHOL] = 1;
    g_init = true;
}

int find(const char *name) {
    if (!name) return -1;
    for (int i = 0; i < OPT_COUNT; ++i)
        if (strcmp(kOpts[i].name, name) == 0) return i;
    return -1;
}

thread_local std::string g_dispatch;
std::atomic<uint64_t> g_gen{0};
}  // namespace

int64_t opt(Opt o) {
    if (!g_init) {
        std::lock_guard<std::mutex> lk(g_mu);
        if (!g_init) init_locked();
    }
    return g_val[o].load(std::memory_order_relaxed);
}

void set_dispatch(const std::string &s) { g_dispatch = s; }

uint64_t options_generation() { return g_gen.load(std::memory_order_relaxed); }

}  // namespace sptk

using namespace sptk;

extern "C" sptk_status sptk_set_option(const char *name, int64_t value) {
    const int i = find(name);
    if (i < 0) return fail(SPTK_EINVAL, std::string("unknown option '") + (name ? name : "") + "'");
    std::lock_guard<std::mutex> lk(g_mu);
    if (!g_init) init_locked();
    if (g_val[i].exchange(value) != value) ++g_gen;
    return SPTK_OK;
}

extern "C" sptk_status sptk_get_option(const char *name, int64_t *value) {
    const int i = find(name);
    if (i < 0 || !value)
        return fail(SPTK_EINVAL, std::string("unknown option '") + (name ? name : "") + "'");
    *value = opt((Opt)i);
    return SPTK_OK;
}

extern "C" sptk_status sptk_reset_options(void) {
    std::lock_guard<std::mutex> lk(g_mu);
    init_locked();
    ++g_gen;
    return SPTK_OK;
}

extern "C" const char *sptk_last_dispatch(void) { return g_dispatch.c_str(); }
