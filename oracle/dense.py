"""Independent pins for the oracle -- TEST INFRASTRUCTURE ONLY.

* ``dense_mttkrp``: the brute force of SURVEY §8(c) -- densify X, form the
  mode-n unfolding X_(n) and the Khatri-Rao product explicitly (Kolda & Bader
  definitions, cited at P:97-98) and multiply.  Shares nothing with
  oracle.c's loop.
* ``planted_mttkrp``: closed form for X = [[mu; B_0..B_{N-1}]] exactly:
  MTTKRP(X, {A}, n) = B_n diag(mu) (Hadamard_{m != n} B_m^T A_m) diag(lambda).
* ``kruskal_dense`` / ``dense_fit``: dense reconstruction of a K-tensor (Eq. (1),
  P:102-121) and the fit 1 - ||X - M|| / ||X|| from it.
"""
from __future__ import annotations

import numpy as np


def densify(dims, idx, vals) -> np.ndarray:
    X = np.zeros(tuple(int(d) for d in dims))
    np.add.at(X, tuple(np.asarray(idx, dtype=np.int64).T), np.asarray(vals, dtype=np.float64))
    return X


def unfold(X: np.ndarray, n: int) -> np.ndarray:
    """Mode-n unfolding X_(n): rows = mode n, columns with lower modes fastest."""
    return np.moveaxis(X, n, 0).reshape(X.shape[n], -1, order="F")


def khatri_rao(B: np.ndarray, C: np.ndarray) -> np.ndarray:
    """Column-wise Kronecker product B (.) C; C's row index varies fastest."""
    IB, R = B.shape
    IC, _ = C.shape
    return (B[:, None, :] * C[None, :, :]).reshape(IB * IC, R)


def krp_excluding(A, n: int) -> np.ndarray:
    """A_{N-1} (.) ... (.) A_{n+1} (.) A_{n-1} (.) ... (.) A_0."""
    K = None
    for m in range(len(A)):
        if m == n:
            continue
        K = np.asarray(A[m], dtype=np.float64) if K is None else khatri_rao(np.asarray(A[m]), K)
    return K


def dense_mttkrp(dims, idx, vals, A, n: int, lam=None) -> np.ndarray:
    V = unfold(densify(dims, idx, vals), n) @ krp_excluding(A, n)
    if lam is not None:
        V = V * np.asarray(lam)[None, :]
    return V


def planted_mttkrp(mu, B, A, n: int, lam=None) -> np.ndarray:
    R = len(mu)
    H = np.ones((R, R))
    for m in range(len(B)):
        if m != n:
            H = H * (np.asarray(B[m]).T @ np.asarray(A[m]))
    V = np.asarray(B[n]) @ (np.diag(mu) @ H)
    if lam is not None:
        V = V * np.asarray(lam)[None, :]
    return V


def kruskal_dense(lam, A) -> np.ndarray:
    N = len(A)
    letters = "abcdefgh"[:N]
    expr = "r," + ",".join(f"{c}r" for c in letters) + "->" + letters
    return np.einsum(expr, np.asarray(lam), *[np.asarray(a) for a in A])


def dense_fit(dims, idx, vals, lam, A) -> float:
    X = densify(dims, idx, vals)
    M = kruskal_dense(lam, A)
    return 1.0 - np.linalg.norm(X - M) / np.linalg.norm(X)
