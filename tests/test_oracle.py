"""Pins for the CPU oracle (no GPU).  Each test ties an oracle function to
something other than itself: a worked example (tests/golden), the dense brute
force (explicit unfolding x explicit Khatri-Rao), the planted-Kruskal closed
form, a library routine for a special case, or an invariant the paper fixes.
"""
import json
import os

import numpy as np
import pytest

import oracle
import synth
from oracle import dense

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def rand_factors(seed, dims, R):
    return [synth.factor(seed, len(dims), m, int(I), R) for m, I in enumerate(dims)]


# ---------------------------------------------------------------- permutation
def test_perm_golden():
    for key in ("perm_singleton", "perm_three"):
        g = GOLD[key]
        p, _ = oracle.perm(np.array(g["idx"]), g["mode"], g["dims"][g["mode"]])
        assert p.tolist() == g["perm"], g["cite"]


@pytest.mark.parametrize("dist", ["uniform", "powerlaw"])
def test_perm_invariants_and_stable_argsort(dist):
    dims = (50, 7, 300)
    idx, _ = synth.tensor(11, dims, 5000, dist)
    for n, I in enumerate(dims):
        p, rowptr = oracle.perm(idx, n, I)
        keys = idx[p, n].astype(np.int64)
        assert np.array_equal(np.sort(p), np.arange(len(p)))          # bijection
        assert np.all(np.diff(keys) >= 0)                               # sorted keys
        ties = np.diff(keys) == 0
        assert np.all(np.diff(p.astype(np.int64))[ties] > 0)            # stable
        # library routine: numpy's stable argsort is the same unique permutation
        assert np.array_equal(p, np.argsort(idx[:, n], kind="stable"))
        assert np.array_equal(rowptr, np.concatenate([[0], np.cumsum(np.bincount(idx[:, n], minlength=I))]))


def test_perm_identity_when_presorted():
    idx = np.array([[0, 5], [0, 1], [1, 1], [3, 0], [3, 2]], dtype=np.uint32)
    p, rp = oracle.perm(idx, 0, 4)
    assert p.tolist() == [0, 1, 2, 3, 4]
    assert rp.tolist() == [0, 2, 3, 3, 5]


def test_perm_rejects_out_of_range():
    with pytest.raises(oracle.OracleError):
        oracle.perm(np.array([[5, 0]]), 0, 3)


# --------------------------------------------------------------------- MTTKRP
def test_mttkrp_golden_single():
    g = GOLD["mttkrp_single"]
    A = [np.ones((d, g["R"])) for d in g["dims"]]
    V = oracle.mttkrp(g["dims"], np.array(g["idx"]), np.array(g["vals"]), A, g["mode"])
    assert V.tolist() == g["V"], g["cite"]


def test_mttkrp_empty_is_zero():
    dims = (4, 5, 6)
    A = rand_factors(3, dims, 3)
    V = oracle.mttkrp(dims, np.zeros((0, 3), np.uint32), np.zeros(0), A, 1)
    assert V.shape == (5, 3) and not V.any()


def test_mttkrp_tiny_config_vs_dense():
    c = synth.CONFIGS["tiny"]
    idx, vals = synth.unique_tensor(c.seed, c.dims, c.nnz)
    A = rand_factors(c.seed_f, c.dims, 8)
    for n in range(3):
        V = oracle.mttkrp(c.dims, idx, vals, A, n)
        assert rel(V, dense.dense_mttkrp(c.dims, idx, vals, A, n)) < 1e-13


@pytest.mark.parametrize("N", [2, 3, 4, 5])
@pytest.mark.parametrize("R", [1, 3, 16, 33])
def test_mttkrp_random_vs_dense(N, R):
    dims = [6, 7, 8, 3, 4][:N]
    idx, vals = synth.tensor(100 + N, dims, 64)             # duplicates allowed (linear)
    A = rand_factors(200 + R, dims, R)
    lam = synth.factor(7, 1, 0, 1, R)[0] + 0.5
    for n in range(N):
        V = oracle.mttkrp(dims, idx, vals, A, n, lam=lam)
        assert rel(V, dense.dense_mttkrp(dims, idx, vals, A, n, lam)) < 1e-13


def test_mttkrp_planted_closed_form():
    dims = (400, 300, 500)
    idx, vals, mu, B = synth.planted_tensor(21, dims, 5, (60, 25, 20))
    assert len(np.unique(idx, axis=0)) == len(idx)          # coordinates unique
    A = rand_factors(22, dims, 5)
    for n in range(3):
        V = oracle.mttkrp(dims, idx, vals, A, n)
        assert rel(V, dense.planted_mttkrp(mu, B, A, n)) < 1e-13


def test_mttkrp_rank1_ones_is_row_histogram():
    dims = (30, 20, 10)
    idx, vals = synth.tensor(5, dims, 3000)
    A = [np.ones((d, 1)) for d in dims]
    for n in range(3):
        V = oracle.mttkrp(dims, idx, vals, A, n)[:, 0]
        np.testing.assert_allclose(V, np.bincount(idx[:, n], weights=vals, minlength=dims[n]),
                                   rtol=1e-13)


def test_mttkrp_linear_and_order_invariant():
    dims = (20, 30, 40)
    idx, vals = synth.tensor(9, dims, 4000)
    A = rand_factors(10, dims, 7)
    V1 = oracle.mttkrp(dims, idx, vals, A, 2)
    V2 = oracle.mttkrp(dims, idx, 3.0 * vals, A, 2)
    assert rel(V2, 3.0 * V1) < 1e-15
    shuf = np.random.default_rng(0).permutation(len(vals))
    V3 = oracle.mttkrp(dims, idx[shuf], vals[shuf], A, 2)
    assert rel(V3, V1) < 1e-14


def test_mttkrp_empty_rows_exactly_zero():
    dims = (50, 4, 4)
    idx, vals = synth.tensor(1, (10, 4, 4), 200)     # rows 10..49 never touched
    A = rand_factors(2, dims, 4)
    V = oracle.mttkrp(dims, idx, vals, A, 0)
    assert not V[10:].any()


def test_mttkrp_rows_omp_long_variants():
    dims = (300, 40, 50)
    idx, vals = synth.tensor(31, dims, 20000, "powerlaw")
    A = rand_factors(32, dims, 16)
    lam = np.linspace(0.5, 2.0, 16)
    for n in range(3):
        V = oracle.mttkrp(dims, idx, vals, A, n, lam=lam)
        rows = np.array([0, 7, dims[n] - 1, 3])
        assert np.array_equal(oracle.mttkrp_rows(dims, idx, vals, A, n, rows, lam=lam), V[rows])
        p, rp = oracle.perm(idx, n, dims[n])
        Vo, nt = oracle.mttkrp_omp(dims, idx, vals, A, n, p, rp, lam=lam)
        assert nt >= 1 and np.array_equal(Vo, V)                     # bit-identical
        Vl = oracle.mttkrp(dims, idx, vals, A, n, lam=lam, acc_long=True)
        assert rel(Vl, V) < 1e-14


# -------------------------------------------------------------- ALS pieces
def test_normalize_golden_and_zero_column():
    g = GOLD["normalize_34"]
    An, lam = oracle.normalize(np.array(g["A"]))
    np.testing.assert_allclose(An, g["A_out"], rtol=1e-15)
    np.testing.assert_allclose(lam, g["lambda"], rtol=1e-15)
    An, lam = oracle.normalize(np.array([[0.0, 1.0], [0.0, 1.0]]))
    assert lam[0] == 0.0 and An[:, 0].tolist() == [1.0, 0.0]


def test_gram_vs_matmul():
    A = synth.factor(4, 3, 0, 50, 8)
    np.testing.assert_allclose(oracle.gram(A), A.T @ A, rtol=1e-13)
    assert np.array_equal(oracle.gram(np.eye(2)), np.eye(2))


def test_chol_solve_cases():
    B = synth.factor(5, 3, 1, 6, 4)
    np.testing.assert_allclose(oracle.chol_solve(np.eye(4), B), B, rtol=1e-15)
    np.testing.assert_allclose(oracle.chol_solve(2 * np.eye(4), B), B / 2, rtol=1e-15)
    Q, _ = np.linalg.qr(synth.factor(6, 3, 2, 4, 4) - 0.5)
    G = Q @ np.diag([4.0, 2.0, 1.0, 0.5]) @ Q.T
    X = oracle.chol_solve(G, B)
    np.testing.assert_allclose(X, np.linalg.solve(G, B.T).T, rtol=1e-12)
    with pytest.raises(oracle.OracleError):
        oracle.chol_solve(np.zeros((3, 3)), np.ones((1, 3)))


def test_chol_solve_ridge_branch():
    """The ridge retry (SURVEY §8(c) CP-ALS step 3.3, DESIGN.md §2 Z11/Z12):
    when Cholesky of Gamma fails, X = B (Gamma + 1e-12 tr(Gamma)/R I)^{-1}.
    Pinned against numpy's LU solve of that explicitly ridged matrix."""
    R = 5
    A = synth.factor(7, 3, 0, 40, R)
    A[:, 3] = 0.0                                  # a zero column: pivot 3 is exactly 0
    G = A.T @ A
    B = synth.factor(8, 3, 1, 6, R) + 0.25
    with np.errstate(all="ignore"):
        assert not np.all(np.linalg.eigvalsh(G) > 0)
    delta = 1e-12 * np.trace(G) / R
    X = oracle.chol_solve(G, B)
    Xr = np.linalg.solve(G + delta * np.eye(R), B.T).T
    # block-diagonal ridged matrix: both solves are well conditioned per block,
    # so they agree to rounding -- including X[:, 3] = B[:, 3] / delta (~1e12)
    np.testing.assert_allclose(X, Xr, rtol=1e-10)
    np.testing.assert_allclose(X[:, 3], B[:, 3] / delta, rtol=1e-14)
    # a wrong ridge (tr(Gamma) instead of tr(Gamma)/R, or no /R at all) is off by R
    assert not np.allclose(X[:, 3], B[:, 3] / (1e-12 * np.trace(G)), rtol=1e-3)
    # rank-deficient but not block-diagonal (two equal columns): the ridged
    # system is ill conditioned (cond ~ 1e12), so pin the residual of the
    # oracle's solve against the ridged matrix instead of forward digits: the
    # right ridge leaves ~u cond(Gr) ~ 1e-4 of ||B||, a ridge off by 10x leaves
    # ~9 delta ||X|| ~ ||B||, twice the ridge ~0.1 ||B||
    A2 = synth.factor(9, 3, 2, 40, R)
    A2[:, 1] = A2[:, 4]
    G2 = A2.T @ A2
    d2 = 1e-12 * np.trace(G2) / R
    X2 = oracle.chol_solve(G2, B)

    def resid(Gx):
        return np.linalg.norm(X2 @ Gx - B) / np.linalg.norm(B)
    assert resid(G2 + d2 * np.eye(R)) <= 1e-3
    assert resid(G2 + 10 * d2 * np.eye(R)) >= 0.1
    assert resid(G2 + 2 * d2 * np.eye(R)) >= 0.05
    assert resid(G2) >= 0.05                      # the unridged matrix


def test_chol_solve_relative_pivot_takes_ridge():
    """DESIGN.md §2 Z23: a pivot d_j <= 1e-12 Gamma_jj is a failure even when
    positive (a numerically singular Gamma, e.g. duplicate CP components).
    Pinned by the 2 x 2 closed form [[a, c], [c, a]]^{-1} = [[a, -c], [-c, a]]
    / (a^2 - c^2): with c = 1 - 2^-46 the pivot is ~2.8e-14 (ridge: a = 1 +
    1e-12); with c = 1 - 2^-34 it is ~1.2e-10 (no ridge: a = 1).  The
    subtraction a - c loses ~4 (resp. ~6) digits, hence the tolerances; the
    unridged and ridged answers differ by ~36x and ~1.017x resp."""
    B = np.array([[1.0, 0.0]])

    def closed(a, c):
        return np.array([[a, -c]]) / ((a - c) * (a + c))

    c = 1.0 - 2.0 ** -46
    G = np.array([[1.0, c], [c, 1.0]])
    X = oracle.chol_solve(G, B)
    np.testing.assert_allclose(X, closed(1.0 + 1e-12, c), rtol=1e-3)
    assert not np.allclose(X, closed(1.0, c), rtol=0.5)   # the plain solve is ~36x larger
    c = 1.0 - 2.0 ** -34
    G = np.array([[1.0, c], [c, 1.0]])
    X = oracle.chol_solve(G, B)
    np.testing.assert_allclose(X, closed(1.0, c), rtol=1e-5)
    assert not np.allclose(X, closed(1.0 + 1e-12, c), rtol=1e-3)  # no ridge here


# ------------------------------------------------------------------- CP-ALS
def _dense_as_sparse(T):
    idx = np.argwhere(T != 0).astype(np.uint32)
    return idx, T[tuple(idx.T.astype(np.int64))]


def test_cp_als_rank1_dense_as_sparse():
    a, b, c = (synth.factor(1, 3, m, I, 1)[:, 0] + 0.1 for m, I in enumerate((5, 6, 7)))
    T = np.einsum("i,j,k->ijk", a, b, c)
    idx, vals = _dense_as_sparse(T)
    init = [synth.factor(2, 3, m, I, 1) for m, I in enumerate((5, 6, 7))]
    out = oracle.cp_als((5, 6, 7), idx, vals, init, 50)
    assert out["fit"] >= 0.999


def test_cp_als_rank4_dense():
    dims = (10, 11, 12)
    F = [synth.factor(3, 3, m, I, 4) + 0.1 for m, I in enumerate(dims)]
    T = dense.kruskal_dense(np.ones(4), F)
    idx, vals = _dense_as_sparse(T)
    init = [synth.factor(4, 3, m, I, 4) for m, I in enumerate(dims)]
    out = oracle.cp_als(dims, idx, vals, init, 100)
    assert out["fit"] >= 0.99


def test_cp_als_planted_sparse_recovery():
    dims = (400, 300, 500)
    idx, vals, mu, B = synth.planted_tensor(21, dims, 5, (60, 25, 20))
    init = rand_factors(23, dims, 5)
    out = oracle.cp_als(dims, idx, vals, init, 60)
    assert out["fit"] > 0.999


def test_cp_als_tiny_monotone_fit_unit_columns_dense_fit():
    c = synth.CONFIGS["tiny"]
    idx, vals = synth.unique_tensor(c.seed, c.dims, c.nnz)
    init = rand_factors(c.seed_f, c.dims, 8)
    out = oracle.cp_als(c.dims, idx, vals, init, 10)
    assert out["iters"] == 10
    assert np.all(np.diff(out["trace"]) >= -1e-12)               # residual non-increasing
    for A in out["A"]:
        np.testing.assert_allclose(np.linalg.norm(A, axis=0), 1.0, rtol=1e-13)
    fd = dense.dense_fit(c.dims, idx, vals, out["lam"], out["A"])
    assert abs(fd - out["fit"]) < 1e-10


def test_cp_als_first_iteration_vs_dense_linear_algebra():
    """One ALS sweep written with dense numpy (unfolding, KRP, np.linalg.solve)."""
    c = synth.CONFIGS["tiny"]
    idx, vals = synth.unique_tensor(c.seed, c.dims, c.nnz)
    A = rand_factors(c.seed_f, c.dims, 8)
    out = oracle.cp_als(c.dims, idx, vals, A, 1)
    A = [a.copy() for a in A]
    for n in range(3):
        V = dense.dense_mttkrp(c.dims, idx, vals, A, n)
        Gam = np.ones((8, 8))
        for m in range(3):
            if m != n:
                Gam *= A[m].T @ A[m]
        An = np.linalg.solve(Gam, V.T).T
        lam = np.linalg.norm(An, axis=0)
        A[n] = An / lam
    for m in range(3):
        assert rel(out["A"][m], A[m]) < 1e-9
    assert rel(out["lam"], lam) < 1e-9


def test_cp_als_tol_stops_early_and_zero_norm():
    dims = (400, 300, 500)
    idx, vals, mu, B = synth.planted_tensor(21, dims, 5, (60, 25, 20))
    out = oracle.cp_als(dims, idx, vals, rand_factors(23, dims, 5), 200, tol=1e-6)
    assert out["iters"] < 200
    with pytest.raises(oracle.OracleError) as e:
        oracle.cp_als((3, 3), np.array([[0, 0]]), np.array([0.0]), [np.ones((3, 2))] * 2, 3)
    assert e.value.code == oracle.EZERONORM


# ------------------------------------------------------------------ duplicates
def test_merge_duplicates_golden_and_dense():
    g = GOLD["dup_merge"]
    io, vo = oracle.merge_duplicates(np.array(g["idx"]), np.array(g["vals"]))
    assert io.tolist() == g["idx_out"] and vo.tolist() == g["vals_out"], g["cite"]
    dims = (5, 4, 3)
    idx, vals = synth.tensor(17, dims, 200)              # 60 cells: many duplicates
    io, vo = oracle.merge_duplicates(idx, vals)
    assert len(np.unique(io, axis=0)) == len(io) < len(idx)
    np.testing.assert_allclose(dense.densify(dims, io, vo), dense.densify(dims, idx, vals),
                               rtol=1e-14)
    # kept order = storage order of first occurrences
    _, first = np.unique(idx, axis=0, return_index=True)
    assert np.array_equal(io, idx[np.sort(first)])
