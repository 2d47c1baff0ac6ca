"""CPU oracle -- TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct implementations of what the hot path computes
(Eq. (2), §5 permutation, textbook CP-ALS).  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline / ``--impl
reference`` leg may import this package.  It shares no code with the CUDA
path and never imports it.

``liboracle.so`` is built from ``oracle.c`` (plain C, fp64, -O2
-ffp-contract=off, OpenMP only in the timing form).  ``dense.py`` holds the
numpy brute force (explicit matricization x explicit Khatri-Rao) and the
planted-Kruskal closed form used to pin this library.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

OK, EINVAL, EZERONORM, ESINGULAR, ENOMEM = 0, -1, -2, -3, -4


class OracleError(RuntimeError):
    def __init__(self, code: int, what: str):
        super().__init__(f"{what}: oracle status {code}")
        self.code = code


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (the checker, not the product)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fopenmp", "-fPIC",
                               "-shared", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        p = C.c_void_p
        i64, i32, dbl = C.c_int64, C.c_int, C.c_double
        L.oracle_perm.argtypes = [i64, i32, p, i32, i64, p, p]
        L.oracle_mttkrp.argtypes = [i32, p, i64, p, p, i64, p, i32, p, i32, p]
        L.oracle_mttkrp_rows.argtypes = [i32, p, i64, p, p, i64, p, i32, p, i32, i64, p, p]
        L.oracle_mttkrp_omp.argtypes = [i32, p, i64, p, p, i64, p, i32, p, p, p, p, p]
        L.oracle_gram.argtypes = [i64, i64, p, p]
        L.oracle_gram.restype = None
        L.oracle_chol_solve.argtypes = [i64, p, i64, p, p]
        L.oracle_normalize.argtypes = [i64, i64, p, p]
        L.oracle_normalize.restype = None
        L.oracle_cp_als.argtypes = [i32, p, i64, p, p, i64, i32, dbl, p, p, p, p, p]
        L.oracle_merge_duplicates.argtypes = [i64, i32, p, p, p, p, p]
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def _idx(idx) -> np.ndarray:
    return np.ascontiguousarray(idx, dtype=np.uint32)


def _factors(A):
    arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in A]
    table = (C.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])
    return arrs, table


def _check(st: int, what: str):
    if st != OK:
        raise OracleError(st, what)


def perm(idx, n: int, In: int):
    """Stable counting-sort permutation of mode n and its row pointers."""
    idx = _idx(idx)
    P, N = idx.shape
    out = np.empty(P, dtype=np.uint32)
    rowptr = np.empty(In + 1, dtype=np.uint32)
    _check(lib().oracle_perm(P, N, _ptr(idx), n, In, _ptr(out), _ptr(rowptr)), "oracle_perm")
    return out, rowptr


def mttkrp(dims, idx, vals, A, n: int, lam=None, acc_long: bool = False) -> np.ndarray:
    """Eq. (2): V = MTTKRP(X, A, n) in fp64, storage order."""
    idx = _idx(idx)
    P, N = idx.shape
    vals = np.ascontiguousarray(vals, dtype=np.float64)
    dims_a = np.ascontiguousarray(dims, dtype=np.int64)
    R = int(np.asarray(A[0]).shape[1])
    arrs, table = _factors(A)
    lam_a = None if lam is None else np.ascontiguousarray(lam, dtype=np.float64)
    V = np.empty((int(dims[n]), R), dtype=np.float64)
    _check(lib().oracle_mttkrp(N, _ptr(dims_a), P, _ptr(idx), _ptr(vals), R, table, n,
                               _ptr(lam_a), int(acc_long), _ptr(V)), "oracle_mttkrp")
    return V


def mttkrp_rows(dims, idx, vals, A, n: int, rows, lam=None, acc_long: bool = False):
    """Eq. (2) for the listed (distinct) rows only."""
    idx = _idx(idx)
    P, N = idx.shape
    vals = np.ascontiguousarray(vals, dtype=np.float64)
    dims_a = np.ascontiguousarray(dims, dtype=np.int64)
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    R = int(np.asarray(A[0]).shape[1])
    arrs, table = _factors(A)
    lam_a = None if lam is None else np.ascontiguousarray(lam, dtype=np.float64)
    out = np.empty((rows.shape[0], R), dtype=np.float64)
    _check(lib().oracle_mttkrp_rows(N, _ptr(dims_a), P, _ptr(idx), _ptr(vals), R, table, n,
                                    _ptr(lam_a), int(acc_long), rows.shape[0], _ptr(rows),
                                    _ptr(out)), "oracle_mttkrp_rows")
    return out


def mttkrp_omp(dims, idx, vals, A, n: int, perm_n, rowptr_n, lam=None):
    """Row-owned OpenMP timing form; returns (V, threads_used)."""
    idx = _idx(idx)
    P, N = idx.shape
    vals = np.ascontiguousarray(vals, dtype=np.float64)
    dims_a = np.ascontiguousarray(dims, dtype=np.int64)
    R = int(np.asarray(A[0]).shape[1])
    arrs, table = _factors(A)
    lam_a = None if lam is None else np.ascontiguousarray(lam, dtype=np.float64)
    V = np.empty((int(dims[n]), R), dtype=np.float64)
    nt = C.c_int(0)
    perm_n = np.ascontiguousarray(perm_n, dtype=np.uint32)
    rowptr_n = np.ascontiguousarray(rowptr_n, dtype=np.uint32)
    _check(lib().oracle_mttkrp_omp(N, _ptr(dims_a), P, _ptr(idx), _ptr(vals), R, table, n,
                                   _ptr(lam_a), _ptr(perm_n), _ptr(rowptr_n), _ptr(V),
                                   C.byref(nt)), "oracle_mttkrp_omp")
    return V, nt.value


def gram(A) -> np.ndarray:
    A = np.ascontiguousarray(A, dtype=np.float64)
    I, R = A.shape
    G = np.empty((R, R))
    lib().oracle_gram(I, R, _ptr(A), _ptr(G))
    return G


def chol_solve(G, B) -> np.ndarray:
    """X = B G^{-1} row by row via Cholesky (ridge retry once)."""
    G = np.ascontiguousarray(G, dtype=np.float64)
    B = np.ascontiguousarray(np.atleast_2d(B), dtype=np.float64)
    X = np.empty_like(B)
    _check(lib().oracle_chol_solve(G.shape[0], _ptr(G), B.shape[0], _ptr(B), _ptr(X)),
           "oracle_chol_solve")
    return X


def normalize(A):
    A = np.array(A, dtype=np.float64, order="C", copy=True)
    I, R = A.shape
    lam = np.empty(R)
    lib().oracle_normalize(I, R, _ptr(A), _ptr(lam))
    return A, lam


def cp_als(dims, idx, vals, init, max_iters: int, tol: float = 0.0):
    """Textbook CP-ALS; returns dict(A, lam, fit, iters, trace)."""
    idx = _idx(idx)
    P, N = idx.shape
    vals = np.ascontiguousarray(vals, dtype=np.float64)
    dims_a = np.ascontiguousarray(dims, dtype=np.int64)
    R = int(np.asarray(init[0]).shape[1])
    arrs = [np.array(a, dtype=np.float64, order="C", copy=True) for a in init]
    table = (C.c_void_p * N)(*[a.ctypes.data for a in arrs])
    lam = np.empty(R)
    fit = C.c_double(0.0)
    iters = C.c_int(0)
    trace = np.zeros(max(max_iters, 1))
    _check(lib().oracle_cp_als(N, _ptr(dims_a), P, _ptr(idx), _ptr(vals), R, max_iters,
                               float(tol), table, _ptr(lam), C.byref(fit), C.byref(iters),
                               _ptr(trace)), "oracle_cp_als")
    return {"A": arrs, "lam": lam, "fit": fit.value, "iters": iters.value,
            "trace": trace[: iters.value]}


def merge_duplicates(idx, vals):
    """Sum duplicate coordinates (first-occurrence position, storage-order sum)."""
    idx = _idx(idx)
    P, N = idx.shape
    vals = np.ascontiguousarray(vals, dtype=np.float64)
    io = np.empty_like(idx)
    vo = np.empty_like(vals)
    Pout = C.c_int64(0)
    _check(lib().oracle_merge_duplicates(P, N, _ptr(idx), _ptr(vals), _ptr(io), _ptr(vo),
                                         C.byref(Pout)), "oracle_merge_duplicates")
    return io[: Pout.value], vo[: Pout.value]
