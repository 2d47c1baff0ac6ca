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
};

static NcclApi &nccl() {
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
    });
    return api;
}

static sptk_status nccl_fail(ncclResult_t r, const char *what) {
    return fail(SPTK_ENCCL, std::string(what) + ": " + nccl().GetErrorString(r));
}

#define SPTK_NCCL(expr)                                                                     \
    do {                                                                                    \
        ncclResult_t _r = (expr);                                                           \
        if (_r != ncclSuccess) return nccl_fail(_r, #expr);                                 \
    } while (0)

sptk_status comm_bcast_rows(sptk_comm c, void *buf, int64_t R, sptk_dtype dt,
                            const int64_t *bounds, cudaStream_t s) {
    NcclApi &api = nccl();
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
    NcclApi &api = nccl();
    if (!api.ok) return fail(SPTK_ENCCL, api.why);
    SPTK_NCCL(api.AllReduce(buf, buf, (size_t)count, ncclFloat64, ncclSum,
                            static_cast<ncclComm_t>(c->nccl), s));
    return SPTK_OK;
}

}  // namespace sptk

using namespace sptk;

extern "C" {

sptk_status sptk_comm_unique_id(void *id128) {
    if (!id128) return fail(SPTK_EINVAL, "id is NULL");
    NcclApi &api = nccl();
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
    NcclApi &api = nccl();
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

sptk_status sptk_comm_destroy(sptk_comm c) {
    if (!c) return SPTK_OK;
    if (c->nccl && nccl().ok) nccl().CommDestroy(static_cast<ncclComm_t>(c->nccl));
    delete c;
    return SPTK_OK;
}

}  // extern "C"
