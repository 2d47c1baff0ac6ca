// comm.cu -- multi-GPU exchange: NCCL over
// NVLink/NVSwitch.  The paper has no distributed layer (P:835 lists it as
// future work); here mode-n rows are sharded in contiguous ranges, so every
// output row is owned by exactly one rank (no cross-GPU atomics) and the
// updated rows are replicated with grouped in-place ncclBroadcast calls (an
// all-gather-v with exact per-rank counts).  NCCL is loaded with dlopen so
// the library loads (and its single-GPU path runs) without it; the same
// libnccl.so.2 torch.distributed already loaded in-process is reused.
#include <dlfcn.h>
#include <stdlib.h>
#include <string.h>
#include <nccl.h>
#ifdef SPTK_NCCL_DEVICE_API
#include <nccl_device.h>
#endif

#include <mutex>

#include "common.cuh"

namespace sptk {

struct NcclApi {
    bool ok = false;
    std::string why;
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Broadcast)(const void *, void *, size_t, ncclDataType_t, int, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t,
                              ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
    // optional: symmetric windows + device communicator (NCCL 2.28, the
    // version whose nccl_device.h comm.cu was compiled against)
    bool sym = false;
    ncclResult_t (*GetVersion)(int *) = nullptr;
    ncclResult_t (*MemAlloc)(void **, size_t) = nullptr;
    ncclResult_t (*MemFree)(void *) = nullptr;
    ncclResult_t (*WindowRegister)(ncclComm_t, void *, size_t, ncclWindow_t *, int) = nullptr;
    ncclResult_t (*WindowDeregister)(ncclComm_t, ncclWindow_t) = nullptr;
#ifdef SPTK_NCCL_DEVICE_API
    ncclResult_t (*DevCommCreate)(ncclComm_t, ncclDevCommRequirements_t const *,
                                  ncclDevComm_t *) = nullptr;
    ncclResult_t (*DevCommDestroy)(ncclComm_t, ncclDevComm_t const *) = nullptr;
    ncclTeam_t (*TeamLsa)(ncclComm_t) = nullptr;
#endif
};

static NcclApi &nccl_api() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            api.why = std::string("dlopen(libnccl.so.2) failed: ") + dlerror();
            return;
        }
#define SYM(name, field)                                                                    \
    api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, name));                      \
    if (!api.field) {                                                                       \
        api.why = std::string("missing NCCL symbol ") + name;                               \
        return;                                                                             \
    }
        SYM("ncclGetUniqueId", GetUniqueId);
        SYM("ncclCommInitRank", CommInitRank);
        SYM("ncclCommDestroy", CommDestroy);
        SYM("ncclBroadcast", Broadcast);
        SYM("ncclAllReduce", AllReduce);
        SYM("ncclGroupStart", GroupStart);
        SYM("ncclGroupEnd", GroupEnd);
        SYM("ncclGetErrorString", GetErrorString);
#undef SYM
        api.ok = true;
#define OPT_SYM(name, field) api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, name))
        OPT_SYM("ncclGetVersion", GetVersion);
        OPT_SYM("ncclMemAlloc", MemAlloc);
        OPT_SYM("ncclMemFree", MemFree);
        OPT_SYM("ncclCommWindowRegister", WindowRegister);
        OPT_SYM("ncclCommWindowDeregister", WindowDeregister);
#ifdef SPTK_NCCL_DEVICE_API
        OPT_SYM("ncclDevCommCreate", DevCommCreate);
        OPT_SYM("ncclDevCommDestroy", DevCommDestroy);
        OPT_SYM("ncclTeamLsa", TeamLsa);
        int v = 0;
        // the window / device-comm structs are read with this build's headers:
        // only the exact version they came from is trusted
        api.sym = api.GetVersion && api.GetVersion(&v) == ncclSuccess && v == NCCL_VERSION_CODE &&
                  api.MemAlloc && api.MemFree && api.WindowRegister && api.WindowDeregister &&
                  api.DevCommCreate && api.DevCommDestroy && api.TeamLsa;
#endif
#undef OPT_SYM
    });
    return api;
}

static sptk_status nccl_fail(ncclResult_t r, const char *what) {
    return fail(SPTK_ENCCL, std::string(what) + ": " + nccl_api().GetErrorString(r));
}

#define SPTK_NCCL(expr)                                                                     \
    do {                                                                                    \
        ncclResult_t _r = (expr);                                                           \
        if (_r != ncclSuccess) return nccl_fail(_r, #expr);                                 \
    } while (0)

sptk_status comm_bcast_rows(sptk_comm c, void *buf, int64_t R, sptk_dtype dt,
                            const int64_t *bounds, cudaStream_t s) {
    NcclApi &api = nccl_api();
    if (!api.ok) return fail(SPTK_ENCCL, api.why);
    const size_t es = dtype_bytes(dt);
    const ncclDataType_t ty = dt == SPTK_F64 ? ncclFloat64 : ncclFloat32;
    ncclComm_t comm = static_cast<ncclComm_t>(c->nccl);
    SPTK_NCCL(api.GroupStart());
    for (int g = 0; g < c->nranks; ++g) {
        char *p = static_cast<char *>(buf) + (size_t)bounds[g] * R * es;
        const size_t n = (size_t)(bounds[g + 1] - bounds[g]) * R;
        ncclResult_t r = api.Broadcast(p, p, n, ty, g, comm, s);
        if (r != ncclSuccess) {
            api.GroupEnd();
            return nccl_fail(r, "ncclBroadcast");
        }
    }
    SPTK_NCCL(api.GroupEnd());
    return SPTK_OK;
}

sptk_status comm_allreduce_f64(sptk_comm c, double *buf, int64_t count, cudaStream_t s) {
    NcclApi &api = nccl_api();
    if (!api.ok) return fail(SPTK_ENCCL, api.why);
    SPTK_NCCL(api.AllReduce(buf, buf, (size_t)count, ncclFloat64, ncclSum,
                            static_cast<ncclComm_t>(c->nccl), s));
    return SPTK_OK;
}

// ------------------------------------------------------------ symmetric memory
static void comm_sym_release(sptk_comm c) {
    NcclApi &api = nccl_api();
    SymMem &m = c->sym;
    if (m.win && api.sym) api.WindowDeregister(static_cast<ncclComm_t>(c->nccl),
                                                static_cast<ncclWindow_t>(m.win));
    if (m.local) {
        if (m.nccl_mem) api.MemFree(m.local);
        else cudaFree(m.local);
    }
    m = SymMem{};
}

// Symmetric buffer of >= bytes on every rank.  With NCCL 2.28: ncclMemAlloc +
// ncclCommWindowRegister(NCCL_WIN_COLL_SYMMETRIC); the window's flat LSA
// mapping gives every rank's copy (stride4G apart), and the device
// communicator's NVLS handle its multicast address.  The exchange mode is the
// minimum over ranks (all-reduce), so every rank takes the same path.
sptk_status comm_sym_reserve(sptk_comm c, size_t bytes, cudaStream_t s) {
    SymMem &m = c->sym;
    if (m.local && m.bytes >= bytes) return SPTK_OK;
    comm_sym_release(c);
    NcclApi &api = nccl_api();
    if (!api.ok) return fail(SPTK_ENCCL, api.why);
    const size_t gran = (size_t)2 << 20;
    const size_t nb = (bytes + gran - 1) / gran * gran;
    const int64_t want = opt(OPT_EXCHANGE);
    ncclComm_t comm = static_cast<ncclComm_t>(c->nccl);
    int cap = 0;  // this rank's capability: 0 broadcast, 1 peer stores, 2 multimem
#ifdef SPTK_NCCL_DEVICE_API
    if (api.sym && want != 0) {
        if (!c->devcomm_tried && (want < 0 || want == 2)) {
            c->devcomm_tried = true;
            ncclDevComm_t *dc = new ncclDevComm_t();
            ncclDevCommRequirements_t req;
            memset(&req, 0, sizeof req);
            req.lsaMultimem = true;
            if (api.DevCommCreate(comm, &req, dc) == ncclSuccess) c->devcomm = dc;
            else delete dc;
        }
        void *p = nullptr;
        ncclWindow_t w = nullptr;
        if (api.MemAlloc(&p, nb) == ncclSuccess) {
            if (api.WindowRegister(comm, p, nb, &w, NCCL_WIN_COLL_SYMMETRIC) == ncclSuccess) {
                m.local = p;
                m.bytes = nb;
                m.win = w;
                m.nccl_mem = true;
                ncclWindow_vidmem wv;
                const ncclTeam_t lsa = api.TeamLsa(comm);
                if (cudaMemcpy(&wv, w, sizeof wv, cudaMemcpyDefault) == cudaSuccess &&
                    lsa.nRanks == c->nranks && c->nranks <= kMaxPeers && wv.lsaRank == c->rank) {
                    for (int r = 0; r < c->nranks; ++r)
                        m.peer[r] = wv.lsaFlatBase + (size_t)r * ((size_t)wv.stride4G << 32);
                    // self-check: our own copy seen through the flat mapping
                    uint64_t a = 0x5157ab1e5eed0001ull, b = 0;
                    bool same = cudaMemcpy(p, &a, 8, cudaMemcpyHostToDevice) == cudaSuccess &&
                                cudaMemcpy(&b, m.peer[c->rank], 8, cudaMemcpyDeviceToHost) ==
                                    cudaSuccess &&
                                a == b;
                    if (same) {
                        m.npeer = c->nranks;
                        cap = 1;
                        ncclDevComm_t *dc = static_cast<ncclDevComm_t *>(c->devcomm);
                        if (dc && dc->lsaMultimem.mcBasePtr) {
                            m.mc = static_cast<char *>(dc->lsaMultimem.mcBasePtr) +
                                   (size_t)wv.mcOffset4K * 4096;
                            cap = 2;
                        }
                    }
                }
                cudaGetLastError();
            } else {
                api.MemFree(p);
            }
        }
    }
#endif
    if (!m.local) {
        SPTK_CUDA(cudaMalloc(&m.local, nb));
        m.bytes = nb;
    }
    if (want >= 0 && want < cap) cap = (int)want;
    // every rank must take the same exchange path: min over ranks
    double *d = nullptr;
    SPTK_CUDA(cudaMalloc(&d, sizeof(double)));
    const double neg = -(double)cap;   // all-reduce has no min: max of -cap
    sptk_status st = SPTK_OK;
    if (cudaMemcpyAsync(d, &neg, sizeof(double), cudaMemcpyHostToDevice, s) != cudaSuccess)
        st = cuda_fail(cudaGetLastError(), "sym exchange agreement");
    NcclApi &a2 = nccl_api();
    if (st == SPTK_OK) {
        ncclResult_t r = a2.AllReduce(d, d, 1, ncclFloat64, ncclMax, comm, s);
        if (r != ncclSuccess) st = nccl_fail(r, "ncclAllReduce(exchange agreement)");
    }
    double agreed = 0.0;
    if (st == SPTK_OK &&
        (cudaMemcpyAsync(&agreed, d, sizeof(double), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
         cudaStreamSynchronize(s) != cudaSuccess))
        st = cuda_fail(cudaGetLastError(), "sym exchange agreement");
    cudaFree(d);
    SPTK_TRY(st);
    m.exchange = (int)(-agreed);
    if (m.exchange < 2) m.mc = nullptr;
    if (m.exchange < 1) m.npeer = 0;
    return SPTK_OK;
}

}  // namespace sptk

using namespace sptk;

extern "C" {

sptk_status sptk_comm_unique_id(void *id128) {
    if (!id128) return fail(SPTK_EINVAL, "id is NULL");
    NcclApi &api = nccl_api();
    if (!api.ok) return fail(SPTK_ENCCL, api.why);
    ncclUniqueId id;
    SPTK_NCCL(api.GetUniqueId(&id));
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId must be 128 bytes");
    memcpy(id128, &id, 128);
    return SPTK_OK;
}

sptk_status sptk_comm_create(const void *id128, int nranks, int rank, sptk_comm *out) {
    if (!id128 || !out || nranks < 1 || rank < 0 || rank >= nranks)
        return fail(SPTK_EINVAL, "comm_create: bad argument");
    *out = nullptr;
    NcclApi &api = nccl_api();
    if (!api.ok) return fail(SPTK_ENCCL, api.why);
    ncclUniqueId id;
    memcpy(&id, id128, 128);
    ncclComm_t comm;
    SPTK_NCCL(api.CommInitRank(&comm, nranks, id, rank));
    sptk_comm c = new sptk_comm_s();
    c->nccl = comm;
    c->nranks = nranks;
    c->rank = rank;
    const char *f = getenv("SPTK_FORCE_SHARDED");
    c->force_sharded = f && *f && *f != '0';
    *out = c;
    return SPTK_OK;
}

sptk_status sptk_comm_exchange(sptk_comm c, int *mode) {
    if (!c || !mode) return fail(SPTK_EINVAL, "comm_exchange: NULL argument");
    *mode = c->sym.local ? c->sym.exchange : -1;
    return SPTK_OK;
}

sptk_status sptk_comm_destroy(sptk_comm c) {
    if (!c) return SPTK_OK;
    if (c->nccl && nccl_api().ok) {
        cudaDeviceSynchronize();
        comm_sym_release(c);
#ifdef SPTK_NCCL_DEVICE_API
        if (c->devcomm) {
            nccl_api().DevCommDestroy(static_cast<ncclComm_t>(c->nccl),
                                  static_cast<ncclDevComm_t *>(c->devcomm));
            delete static_cast<ncclDevComm_t *>(c->devcomm);
        }
#endif
        nccl_api().CommDestroy(static_cast<ncclComm_t>(c->nccl));
    }
    delete c;
    return SPTK_OK;
}

}  // extern "C"
