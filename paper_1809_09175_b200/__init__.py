"""Thin Python binding of libsptk.so (C ABI in include/sptk.h).

Argument marshalling only: every step of the path runs in the library's
CUDA kernels.  There is no CPU fallback -- if libsptk.so is missing or fails
to load, every call raises.  Python names are the C names without the
``sptk_`` prefix.  Tensors are torch tensors (device or pinned/pageable host)
or numpy arrays (host); their ``data_ptr`` is passed straight through.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# SPTK_LIB overrides the in-tree library (A/B measurements of two builds)
LIB_PATH = os.environ.get("SPTK_LIB") or os.path.join(_HERE, "libsptk.so")

F32, F64 = 1, 2
IDX_I64, IDX_U32 = 1, 2
CREATE_DEFAULT, CREATE_PERM_GATHER, CREATE_DETERMINISTIC = 0, 2, 4
CREATE_DUP_SUM, CREATE_DUP_ERROR = 8, 16
STATUS = {0: "OK", 1: "EINVAL", 2: "ERANGE", 3: "EDUP", 4: "ENOPERM", 5: "ENOMEM",
          6: "ECUDA", 7: "ENCCL", 8: "ESINGULAR", 9: "EZERONORM", 10: "EUNSUPPORTED"}
CODES = {v: k for k, v in STATUS.items()}


class SptkError(RuntimeError):
    def __init__(self, code: int, fn: str, msg: str):
        super().__init__(f"{fn}: SPTK_{STATUS.get(code, code)}: {msg}")
        self.code = code
        self.name = STATUS.get(code, str(code))


_lib = None

# (name, argtypes, restype)
_P, _I, _I64, _U64, _D, _U = C.c_void_p, C.c_int, C.c_int64, C.c_uint64, C.c_double, C.c_uint
_SIGS = [
    ("sptk_version", [], C.c_char_p),
    ("sptk_last_error", [], C.c_char_p),
    ("sptk_sptensor_create", [_I, _P, _I64, _P, _I, _P, _I, _U, _P, _P], _I),
    ("sptk_sptensor_destroy", [_P], _I),
    ("sptk_sptensor_info", [_P, _P, _P, _P, _P], _I),
    ("sptk_sptensor_device_bytes", [_P, _P], _I),
    ("sptk_sptensor_set_shard", [_P, _I, _I], _I),
    ("sptk_build_perm", [_P, _I, _P], _I),
    ("sptk_get_perm", [_P, _I, _P, _P], _I),
    ("sptk_get_rowptr", [_P, _I, _P, _P], _I),
    ("sptk_mttkrp", [_P, _I, _I64, _P, _P, _P, _P, _P], _I),
    ("sptk_mttkrp_rows", [_P, _I, _I64, _P, _P, _P, _I64, _I64, _P], _I),
    ("sptk_mttkrp_atomic", [_P, _I, _I64, _P, _P, _P, _P], _I),
    ("sptk_cp_als", [_P, _I64, _I, _D, _U64, _P, _P, _P, _P, _P, _P, _P, _P], _I),
    ("sptk_comm_unique_id", [_P], _I),
    ("sptk_comm_create", [_P, _I, _I, _P], _I),
    ("sptk_comm_destroy", [_P], _I),
    ("sptk_comm_exchange", [_P, _P], _I),
    ("sptk_partition_rows", [_P, _I64, _I, _P], _I),
    ("sptk_profile_enable", [_I], _I),
    ("sptk_profile_reset", [], _I),
    ("sptk_profile_read", [_P, _P, _P], _I),
    ("sptk_set_tuning", [_I, _I64], _I),
    ("sptk_set_option", [C.c_char_p, _I64], _I),
    ("sptk_get_option", [C.c_char_p, _P], _I),
    ("sptk_reset_options", [], _I),
    ("sptk_last_dispatch", [], C.c_char_p),
]
EXPORTS = [s[0] for s in _SIGS]


def lib():
    """Load libsptk.so (raises if it is missing: no fallback path exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} not built: run `python -m paper_1809_09175_b200.build`"
                               " (there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, args, res in _SIGS:
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _lib = L
    return _lib


def _check(st: int, fn: str):
    if st != 0:
        raise SptkError(st, fn, lib().sptk_last_error().decode())


def version() -> str:
    return lib().sptk_version().decode()


# ------------------------------------------------------------------ marshalling
def _ptr(x):
    """Raw address of a torch tensor / numpy array (None -> NULL)."""
    if x is None:
        return None
    if isinstance(x, np.ndarray):
        if not x.flags["C_CONTIGUOUS"]:
            raise ValueError("numpy array must be C-contiguous")
        return x.ctypes.data
    if hasattr(x, "data_ptr"):
        if not x.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return x.data_ptr()
    raise TypeError(f"unsupported buffer type {type(x)}")


def _dtype_code(x) -> int:
    name = str(getattr(x, "dtype", ""))
    if name.endswith("float64"):
        return F64
    if name.endswith("float32"):
        return F32
    raise TypeError(f"values must be float32 or float64, got {name}")


def _idx_code(x) -> int:
    name = str(getattr(x, "dtype", ""))
    if name.endswith("int64"):
        return IDX_I64
    if name.endswith("uint32") or name.endswith("int32"):
        return IDX_U32
    raise TypeError(f"indices must be int64 or (u)int32, got {name}")


def _stream(stream):
    if stream is not None:
        return stream if isinstance(stream, int) else stream.cuda_stream
    try:
        import torch
        if torch.cuda.is_available():
            return torch.cuda.current_stream().cuda_stream
    except Exception:  # pragma: no cover
        pass
    return None


class SpTensor:
    """Owning wrapper of an sptk_tensor handle."""

    def __init__(self, handle: int, dims, nnz: int, dtype: int, device: int = 0):
        self.handle = C.c_void_p(handle)
        self.dims = tuple(int(d) for d in dims)
        self.nnz = int(nnz)
        self.dtype = dtype
        self.device = device   # CUDA device the handle's memory lives on

    @property
    def N(self) -> int:
        return len(self.dims)

    def close(self):
        if self.handle and self.handle.value:
            lib().sptk_sptensor_destroy(self.handle)
            self.handle = C.c_void_p(0)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _current_device() -> int:
    try:
        import torch
        if torch.cuda.is_available():
            return torch.cuda.current_device()
    except Exception:  # pragma: no cover
        pass
    return 0


def _is_cuda(x) -> bool:
    return bool(getattr(x, "is_cuda", False))


def _check_buf(t: "SpTensor", x, shape, what: str, device_only: bool):
    """Validate one factor / output / lambda buffer before its raw address
    crosses the C ABI (which cannot see shapes or dtypes): exact shape, the
    tensor's dtype, C-contiguous, and -- for device buffers -- the tensor's
    device.  device_only: host buffers are refused (mttkrp takes device
    pointers only)."""
    if x is None:
        raise ValueError(f"{what} is None")
    got = tuple(int(d) for d in getattr(x, "shape", ()))
    if got != tuple(shape):
        raise ValueError(f"{what}: shape {got}, expected {tuple(shape)}")
    try:
        code = _dtype_code(x)
    except TypeError as e:
        raise ValueError(f"{what}: {e}") from None
    if code != t.dtype:
        raise ValueError(f"{what}: dtype {getattr(x, 'dtype', '?')} does not match the tensor's "
                         f"{'float64' if t.dtype == F64 else 'float32'}")
    contig = x.flags["C_CONTIGUOUS"] if isinstance(x, np.ndarray) else x.is_contiguous()
    if not contig:
        raise ValueError(f"{what}: must be C-contiguous")
    if _is_cuda(x):
        if x.device.index != t.device:
            raise ValueError(f"{what}: on cuda:{x.device.index}, the tensor lives on cuda:{t.device}")
    elif device_only:
        raise ValueError(f"{what}: must be a CUDA tensor (device pointer)")


def _check_factors(t: "SpTensor", factors, R: int, what: str, skip_mode=None,
                   device_only: bool = True):
    if len(factors) != t.N:
        raise ValueError(f"{what}: {len(factors)} matrices for a {t.N}-way tensor")
    for m, a in enumerate(factors):
        if m == skip_mode and a is None:
            continue
        _check_buf(t, a, (t.dims[m], R), f"{what}[{m}]", device_only)


def _check_mttkrp_args(t: "SpTensor", mode: int, factors, out, lam):
    if not 0 <= mode < t.N:
        raise ValueError(f"mode {mode} outside [0, {t.N})")
    if len(factors) != t.N:
        raise ValueError(f"factors: {len(factors)} matrices for a {t.N}-way tensor")
    R = int(out.shape[1]) if getattr(out, "shape", None) is not None and len(out.shape) == 2 else -1
    if R < 1:
        raise ValueError("out must be a 2-D (I_mode, R) buffer")
    _check_buf(t, out, (t.dims[mode], R), "out", True)
    _check_factors(t, factors, R, "factors", skip_mode=mode)
    if lam is not None:
        _check_buf(t, lam, (R,), "lam", True)
    return R


# ------------------------------------------------------------------ API
def sptensor_create(dims, idx, vals, stream=None, perm_gather: bool = False,
                    deterministic: bool = False, duplicates: str = "allow") -> SpTensor:
    """perm_gather=True keeps the paper's literal traversal (gather records
    through perm_n) instead of materialising permuted copies at build_perm;
    deterministic=True makes MTTKRP / CP-ALS bit-reproducible; duplicates is
    "allow" (default), "sum" (merge) or "error" (SPTK_EDUP)."""
    dup = {"allow": 0, "sum": CREATE_DUP_SUM, "error": CREATE_DUP_ERROR}[duplicates]
    dims_a = np.ascontiguousarray(dims, dtype=np.int64)
    nnz = int(vals.shape[0])
    if nnz > 0 and tuple(idx.shape) != (nnz, len(dims_a)):
        raise ValueError(f"idx shape {tuple(idx.shape)} != ({nnz}, {len(dims_a)})")
    out = C.c_void_p(0)
    dt = _dtype_code(vals)
    _check(lib().sptk_sptensor_create(len(dims_a), dims_a.ctypes.data, nnz, _ptr(idx) if nnz else None,
                                      _idx_code(idx), _ptr(vals) if nnz else None, dt,
                                      (CREATE_PERM_GATHER if perm_gather else 0)
                                      | (CREATE_DETERMINISTIC if deterministic else 0) | dup,
                                      _stream(stream), C.byref(out)), "sptensor_create")
    tt = SpTensor(out.value, dims_a, nnz, dt, _current_device())
    if dup:
        tt.nnz = sptensor_info(tt)["nnz"]
    return tt


def sptensor_info(t: SpTensor):
    n = C.c_int(0)
    dims = np.zeros(6, dtype=np.int64)
    nnz = C.c_int64(0)
    dt = C.c_int(0)
    _check(lib().sptk_sptensor_info(t.handle, C.byref(n), dims.ctypes.data, C.byref(nnz),
                                    C.byref(dt)), "sptensor_info")
    return {"nmodes": n.value, "dims": tuple(dims[: n.value].tolist()), "nnz": nnz.value,
            "dtype": dt.value}


def sptensor_device_bytes(t: SpTensor) -> int:
    b = C.c_int64(0)
    _check(lib().sptk_sptensor_device_bytes(t.handle, C.byref(b)), "sptensor_device_bytes")
    return b.value


def sptensor_set_shard(t: SpTensor, nranks: int, rank: int):
    """This handle serves rank `rank` of `nranks` row-range shards: the permuted
    copies built afterwards hold only this rank's rows (1/nranks of the memory)."""
    _check(lib().sptk_sptensor_set_shard(t.handle, nranks, rank), "sptensor_set_shard")


def build_perm(t: SpTensor, mode: int = -1, stream=None):
    _check(lib().sptk_build_perm(t.handle, mode, _stream(stream)), "build_perm")


def get_perm(t: SpTensor, mode: int, out, stream=None):
    _check(lib().sptk_get_perm(t.handle, mode, _ptr(out), _stream(stream)), "get_perm")
    return out


def get_rowptr(t: SpTensor, mode: int, out, stream=None):
    _check(lib().sptk_get_rowptr(t.handle, mode, _ptr(out), _stream(stream)), "get_rowptr")
    return out


def _ptr_table(arrs):
    return (C.c_void_p * len(arrs))(*[_ptr(a) for a in arrs])


def mttkrp(t: SpTensor, mode: int, factors, out, lam=None, comm=None, stream=None):
    """out <- MTTKRP(X, factors, mode) (Eq. (2)); factors[mode] may be None."""
    R = _check_mttkrp_args(t, mode, factors, out, lam)
    table = _ptr_table(factors)
    _check(lib().sptk_mttkrp(t.handle, mode, R, table, _ptr(lam), _ptr(out),
                             comm.handle if comm is not None else None, _stream(stream)),
           "mttkrp")
    return out


def mttkrp_atomic(t: SpTensor, mode: int, factors, out, lam=None, stream=None):
    """The paper's atomic-per-nonzero MTTKRP (VerA/VerB): storage order, no perm."""
    R = _check_mttkrp_args(t, mode, factors, out, lam)
    _check(lib().sptk_mttkrp_atomic(t.handle, mode, R, _ptr_table(factors), _ptr(lam), _ptr(out),
                                    _stream(stream)), "mttkrp_atomic")
    return out


def mttkrp_rows(t: SpTensor, mode: int, factors, out, row_begin: int, row_end: int, lam=None,
                stream=None):
    """out[row_begin:row_end] <- those rows of MTTKRP(X, factors, mode)."""
    R = _check_mttkrp_args(t, mode, factors, out, lam)
    _check(lib().sptk_mttkrp_rows(t.handle, mode, R, _ptr_table(factors), _ptr(lam), _ptr(out),
                                  row_begin, row_end, _stream(stream)), "mttkrp_rows")
    return out


def cp_als(t: SpTensor, R: int, max_iters: int, factors_out, tol: float = 0.0, seed: int = 0,
           init=None, lambda_out=None, comm=None, stream=None, trace: bool = True):
    """Runs CP-ALS; factors_out (and init) are lists of per-mode buffers.
    Returns dict(fit, iters, trace).  Buffers may be device (the tensor's
    device) or host; each must be (I_m, R) of the tensor's dtype."""
    if int(R) < 1:
        raise ValueError("R must be >= 1")
    _check_factors(t, factors_out, R, "factors_out", device_only=False)
    if init is not None:
        _check_factors(t, init, R, "init", device_only=False)
    if lambda_out is not None:
        _check_buf(t, lambda_out, (R,), "lambda_out", False)
    fit = C.c_double(0.0)
    iters = C.c_int(0)
    tr = np.zeros(max(max_iters, 1), dtype=np.float64)
    init_t = _ptr_table(init) if init is not None else None
    _check(lib().sptk_cp_als(t.handle, R, max_iters, float(tol), int(seed), init_t,
                             _ptr_table(factors_out), _ptr(lambda_out), C.byref(fit),
                             C.byref(iters), tr.ctypes.data if trace else None,
                             comm.handle if comm is not None else None, _stream(stream)),
           "cp_als")
    return {"fit": fit.value, "iters": iters.value, "trace": tr[: iters.value]}


class Comm:
    def __init__(self, handle: int, nranks: int, rank: int):
        self.handle = C.c_void_p(handle)
        self.nranks = nranks
        self.rank = rank

    def close(self):
        if self.handle and self.handle.value:
            lib().sptk_comm_destroy(self.handle)
            self.handle = C.c_void_p(0)


def comm_unique_id() -> bytes:
    buf = (C.c_char * 128)()
    _check(lib().sptk_comm_unique_id(buf), "comm_unique_id")
    return bytes(buf)


def comm_create(uid: bytes, nranks: int, rank: int) -> Comm:
    out = C.c_void_p(0)
    buf = (C.c_char * 128).from_buffer_copy(uid)
    _check(lib().sptk_comm_create(buf, nranks, rank, C.byref(out)), "comm_create")
    return Comm(out.value, nranks, rank)


def comm_exchange(comm: Comm) -> int:
    """Row-exchange mode of the sharded CP-ALS on this communicator: 2 NVLS
    multimem stores, 1 peer stores, 0 NCCL broadcasts, -1 not decided yet."""
    v = C.c_int(0)
    _check(lib().sptk_comm_exchange(comm.handle, C.byref(v)), "comm_exchange")
    return v.value


def comm_from_process_group(group=None) -> Comm:
    """Bootstrap an sptk communicator from an initialised torch.distributed
    group (used only to broadcast the 128-byte NCCL id)."""
    import torch
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    uid = comm_unique_id() if rank == 0 else bytes(128)
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" \
        else torch.device("cpu")
    buf = torch.tensor(list(uid), dtype=torch.uint8, device=dev)
    dist.broadcast(buf, 0, group=group)
    return comm_create(bytes(buf.cpu().tolist()), world, rank)


def partition_rows(rowptr, nranks: int) -> np.ndarray:
    """Host-only row-range split (no GPU needed)."""
    rp = np.ascontiguousarray(rowptr, dtype=np.uint32)
    bounds = np.zeros(nranks + 1, dtype=np.int64)
    _check(lib().sptk_partition_rows(rp.ctypes.data, rp.shape[0] - 1, nranks, bounds.ctypes.data),
           "partition_rows")
    return bounds


def set_tuning(variant: int = -1, run: int = 0):
    """variant: 0 per-group, 1 warp-cooperative, -1 keep, -2 automatic; run: 0 keep, -2 adaptive."""
    _check(lib().sptk_set_tuning(variant, run), "set_tuning")


def set_option(name: str, value: int):
    """Process-wide launch option (names and meaning in include/sptk.h)."""
    _check(lib().sptk_set_option(name.encode(), int(value)), "set_option")


def get_option(name: str) -> int:
    v = C.c_int64(0)
    _check(lib().sptk_get_option(name.encode(), C.byref(v)), "get_option")
    return v.value


def reset_options():
    _check(lib().sptk_reset_options(), "reset_options")


def last_dispatch() -> str:
    """Traversal of the last MTTKRP call on this thread (e.g. "slice V4")."""
    return lib().sptk_last_dispatch().decode()


class options:
    """Context manager: ``with sp.options(slice=0, variant=1): ...`` sets the
    options and restores their previous values on exit."""

    def __init__(self, **kw):
        self.kw = kw
        self.prev = {}

    def __enter__(self):
        for k, v in self.kw.items():
            self.prev[k] = get_option(k)
            set_option(k, v)
        return self

    def __exit__(self, *exc):
        for k, v in self.prev.items():
            set_option(k, v)
        return False


def profile_enable(on: bool = True):
    _check(lib().sptk_profile_enable(int(on)), "profile_enable")


def profile_reset():
    _check(lib().sptk_profile_reset(), "profile_reset")


def profile_read():
    ms = C.c_double(0)
    n = C.c_int64(0)
    k = C.c_int64(0)
    _check(lib().sptk_profile_read(C.byref(ms), C.byref(n), C.byref(k)), "profile_read")
    return {"mttkrp_ms": ms.value, "mttkrp_launches": n.value, "kernel_launches": k.value}
