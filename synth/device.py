"""Device-side generator (libsynth.so, built from synth/gen.cu): writes the
same inputs as the numpy functions in synth/__init__.py straight into CUDA
memory (torch tensors).  Input generation only -- no method arithmetic."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import POW2_COEFFS, PowerLawParams

_LIB = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libsynth.so")
_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB):
            raise RuntimeError(f"{_LIB} missing: run `python -m paper_1809_09175_b200.build`")
        L = C.CDLL(_LIB)
        p, u64, i, i64, d = C.c_void_p, C.c_uint64, C.c_int, C.c_int64, C.c_double
        L.synth_coords.argtypes = [u64, i, i, C.c_uint32, u64, i64, i, d, u64, u64, p, p, p]
        L.synth_values.argtypes = [u64, i, u64, i64, i, p, p]
        L.synth_factor.argtypes = [u64, i, i, i64, i64, i, p, p]
        L.synth_coords_at.argtypes = [u64, i, C.c_uint32, p, i64, i, d, u64, u64, p, p, p]
        L.synth_values_at.argtypes = [u64, i, p, i64, p, p]
        _lib = L
    return _lib


_COEFFS = np.ascontiguousarray(POW2_COEFFS)


def _stream():
    import torch
    return torch.cuda.current_stream().cuda_stream


def tensor(seed: int, dims, P: int, dist: str = "uniform", i0: int = 0, dtype=None,
           device="cuda"):
    """(idx uint32-as-int32 [P,N] on device, vals [P] on device)."""
    import torch
    dtype = dtype or torch.float64
    N = len(dims)
    idx = torch.empty((P, N), dtype=torch.int32, device=device)
    vals = torch.empty(P, dtype=dtype, device=device)
    if P == 0:
        return idx, vals
    for m, I in enumerate(dims):
        pl = PowerLawParams.for_dim(int(I)) if dist == "powerlaw" else PowerLawParams(0.0, 0, 0)
        st = lib().synth_coords(seed, m, N, int(I), i0, P, 1 if dist == "powerlaw" else 0,
                                pl.L, pl.a, pl.b, _COEFFS.ctypes.data, idx.data_ptr(), _stream())
        if st:
            raise RuntimeError(f"synth_coords failed: cuda error {st}")
    st = lib().synth_values(seed, N, i0, P, int(dtype == torch.float32), vals.data_ptr(), _stream())
    if st:
        raise RuntimeError(f"synth_values failed: cuda error {st}")
    return idx, vals


def factor(seed_f: int, N: int, m: int, I: int, R: int, dtype=None, device="cuda"):
    import torch
    dtype = dtype or torch.float64
    out = torch.empty((I, R), dtype=dtype, device=device)
    st = lib().synth_factor(seed_f, N, m, I, R, int(dtype == torch.float32), out.data_ptr(),
                            _stream())
    if st:
        raise RuntimeError(f"synth_factor failed: cuda error {st}")
    return out


def coords_at(seed: int, mode: int, I: int, ids, dist: str = "uniform"):
    """Mode-`mode` coordinates of the nonzeros with generation counters `ids`
    (a CUDA int32 tensor holding uint32 counters) -> CUDA int32 tensor."""
    import torch
    out = torch.empty_like(ids)
    pl = PowerLawParams.for_dim(int(I)) if dist == "powerlaw" else PowerLawParams(0.0, 0, 0)
    st = lib().synth_coords_at(seed, mode, int(I), ids.data_ptr(), ids.numel(),
                               1 if dist == "powerlaw" else 0, pl.L, pl.a, pl.b,
                               _COEFFS.ctypes.data, out.data_ptr(), _stream())
    if st:
        raise RuntimeError(f"synth_coords_at failed: cuda error {st}")
    return out


def values_at(seed: int, N: int, ids):
    """fp64 values of the nonzeros with generation counters `ids`."""
    import torch
    out = torch.empty(ids.numel(), dtype=torch.float64, device=ids.device)
    st = lib().synth_values_at(seed, N, ids.data_ptr(), ids.numel(), out.data_ptr(), _stream())
    if st:
        raise RuntimeError(f"synth_values_at failed: cuda error {st}")
    return out


def int_values_from(vals):
    """Integer values 1 + floor(4u) from device values x = 1 - u (fp64; 1 - x is
    exactly u for u a multiple of 2^-53 in [0,1)) -- same integers as
    ``synth.int_values``."""
    from . import INT_VALUE_LEVELS, int_from_unit
    return int_from_unit(1.0 - vals.double(), INT_VALUE_LEVELS)


def int_factor(seed_f: int, N: int, m: int, I: int, R: int, dtype=None, device="cuda"):
    """Integer factor 1 + floor(3u) (same integers as ``synth.int_factor``)."""
    import torch
    from . import INT_FACTOR_LEVELS, int_from_unit
    u = factor(seed_f, N, m, I, R, dtype=torch.float64, device=device)
    return int_from_unit(u, INT_FACTOR_LEVELS).to(dtype or torch.float64)
