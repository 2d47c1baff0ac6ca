"""GPU parity tests: the CUDA path (through the C ABI) against the CPU oracle
on the same seeded inputs.

Bars (BASELINE.json north_star): permutations bit-exact; MTTKRP relative
Frobenius error <= 1e-12 (fp64) / <= 1e-5 (fp32, oracle in fp64 on the
fp32-rounded inputs); CP-ALS trajectory within the DESIGN.md §5 tolerances.
"""
import os

import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = {torch.float64: 1e-12, torch.float32: 1e-5}


@pytest.fixture(scope="module")
def sp():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import paper_1809_09175_b200 as sp
    sp.lib()          # raises if the extension is missing: no fallback
    return sp


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def dev(x, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    return t.to(dtype) if dtype is not None else t


def make(sp, dims, idx, vals, dtype=torch.float64, perm_gather=False):
    return sp.sptensor_create(dims, dev(idx.astype(np.int64)), dev(vals, dtype),
                              perm_gather=perm_gather)


def factors_np(seed, dims, R, dtype=np.float64):
    return [synth.factor(seed, len(dims), m, int(I), R).astype(dtype) for m, I in enumerate(dims)]


def gpu_mttkrp(sp, t, n, A_np, R, dtype, lam=None, offset=0):
    """Factors passed as device tensors; offset > 0 shifts the base pointer
    (a view into a larger buffer) to exercise the unaligned/generic path."""
    A_dev = []
    for a in A_np:
        if offset:
            buf = torch.zeros(a.size + offset, dtype=dtype, device="cuda")
            buf[offset:] = dev(a.reshape(-1), dtype)
            A_dev.append(buf[offset:].view(a.shape))
        else:
            A_dev.append(dev(a, dtype))
    out = torch.full((t.dims[n], R), float("nan"), dtype=dtype, device="cuda")
    lam_d = dev(lam, dtype) if lam is not None else None
    sp.mttkrp(t, n, A_dev, out, lam=lam_d)
    torch.cuda.synchronize()
    return out.double().cpu().numpy()


def gpu_perm(sp, t, n):
    p = torch.empty(max(t.nnz, 1), dtype=torch.int32, device="cuda")
    rp = torch.empty(t.dims[n] + 1, dtype=torch.int32, device="cuda")
    sp.get_perm(t, n, p)
    sp.get_rowptr(t, n, rp)
    return (p.cpu().numpy().view(np.uint32)[: t.nnz], rp.cpu().numpy().view(np.uint32))


# ------------------------------------------------------------------ perms
@pytest.mark.parametrize("case", [
    ("uniform", (100, 80, 60), 2000),
    ("uniform", (300, 70000, 5), 3 * 4096 + 17),          # 1, 3 (17 bits -> 3 passes), 1 pass
    ("powerlaw", (532000, 1400, 2), 50000),
    ("uniform", (1, 7, 2), 999),                          # I_n = 1 (0 key bits)
    ("uniform", (3, 4), 1),
    ("uniform", (4000, 2, 3), 60 * 4096 + 5),              # many tiles: look-back chains
    ("uniform", (5000, 300, 7), 700 * 4096 + 3),           # > 2 tiles per persistent block
])
@pytest.mark.parametrize("sort", [{}, {"sort_v1": 1}])
def test_perm_bitexact(sp, case, sort):
    """Both radix downsweeps (the default, the round-1 kernel) give the
    oracle's stable order, incl. misaligned key slices (P % 4 != 0) and
    partial last tiles."""
    dist, dims, P = case
    idx, vals = synth.tensor(41, dims, P, dist)
    for keep in (1, 0):
        with sp.options(keep_keys=keep, **sort):
            t = make(sp, dims, idx, vals)
            sp.build_perm(t, -1)            # sorts from the keys the ingest pass emitted
            for n in range(len(dims)):
                p, rp = gpu_perm(sp, t, n)
                po, rpo = oracle.perm(idx, n, dims[n])
                assert np.array_equal(p, po), f"mode {n}"
                assert np.array_equal(rp, rpo), f"mode {n}"
            # re-sort: from the resident keys (keep 1) or extracted from the records (keep 0)
            sp.build_perm(t, 0)
            p, rp = gpu_perm(sp, t, 0)
            assert np.array_equal(p, oracle.perm(idx, 0, dims[0])[0])
            t.close()


def test_perm_golden_and_empty(sp):
    t = make(sp, (3, 1), np.array([[2, 0], [0, 0], [1, 0]]), np.array([1.0, 2.0, 3.0]))
    sp.build_perm(t, 0)
    assert gpu_perm(sp, t, 0)[0].tolist() == [1, 2, 0]
    e = sp.sptensor_create((4, 5), torch.zeros((0, 2), dtype=torch.int64, device="cuda"),
                           torch.zeros(0, dtype=torch.float64, device="cuda"))
    sp.build_perm(e, -1)
    assert gpu_perm(sp, e, 1)[1].tolist() == [0] * 6
    out = torch.full((4, 3), 7.0, dtype=torch.float64, device="cuda")
    A = [torch.rand(4, 3, dtype=torch.float64, device="cuda"),
         torch.rand(5, 3, dtype=torch.float64, device="cuda")]
    sp.mttkrp(e, 0, A, out)
    assert not out.any()


# ------------------------------------------------------------------ MTTKRP
@pytest.mark.parametrize("layout", ["sorted", "perm_gather"])
@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
@pytest.mark.parametrize("N,R", [(3, 8), (3, 16), (3, 64), (3, 128), (3, 256), (4, 16),
                                 (5, 16), (3, 24), (4, 32),
                                 # R not a multiple of 32 bytes: narrower lane vectors
                                 (3, 1), (3, 10), (3, 17), (3, 20), (4, 6), (5, 13), (3, 100),
                                 (3, 258)])
def test_mttkrp_fast_path_parity(sp, layout, dtype, N, R):
    dims = [57, 1203, 311, 40, 9][:N]
    P = 5 * 4096 + 123
    idx, vals = synth.tensor(1000 + N, dims, P, "uniform")
    npd = np.float64 if dtype == torch.float64 else np.float32
    vals = vals.astype(npd)
    A = factors_np(2000 + R, dims, R, npd)
    lam = np.linspace(0.5, 1.5, R).astype(npd)
    t = make(sp, dims, idx, vals, dtype, perm_gather=layout == "perm_gather")
    sp.build_perm(t, -1)
    for n in range(N):
        for L in (None, lam):
            V = gpu_mttkrp(sp, t, n, A, R, dtype, lam=L)
            Vo = oracle.mttkrp(dims, idx, vals.astype(np.float64), [a.astype(np.float64) for a in A],
                               n, lam=None if L is None else L.astype(np.float64))
            assert rel(V, Vo) <= TOL[dtype], (n, L is None)


@pytest.mark.parametrize("layout", ["sorted", "perm_gather"])
@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
@pytest.mark.parametrize("dims,R,offset", [
    ((40, 1000), 1, 0), ((40, 1000), 3, 0), ((7, 9, 11, 3, 5, 4), 17, 0),   # N = 2, 6 generic
    ((33,), 5, 0),                                                          # N = 1: per-row sums
    ((57, 1203, 311), 33, 0), ((57, 1203, 311), 130, 0),                    # odd R, col tiles
    ((57, 1203, 311), 16, 1),                                               # unaligned factors
])
def test_mttkrp_generic_path_parity(sp, layout, dtype, dims, R, offset):
    P = 3 * 4096 + 5
    idx, vals = synth.tensor(77, dims, P, "uniform")
    npd = np.float64 if dtype == torch.float64 else np.float32
    vals = vals.astype(npd)
    A = factors_np(78, dims, R, npd)
    t = make(sp, dims, idx, vals, dtype, perm_gather=layout == "perm_gather")
    sp.build_perm(t, -1)
    for n in range(len(dims)):
        V = gpu_mttkrp(sp, t, n, A, R, dtype, offset=offset)
        Vo = oracle.mttkrp(dims, idx, vals.astype(np.float64), [a.astype(np.float64) for a in A], n)
        assert rel(V, Vo) <= TOL[dtype], n


@pytest.mark.parametrize("dtype,R", [(torch.float64, 16), (torch.float32, 16),
                                     (torch.float64, 8), (torch.float32, 32),
                                     (torch.float64, 10), (torch.float32, 13)])
def test_mttkrp_slice_traversal(sp, dtype, R):
    """Rows long enough for the slice traversal (mode 0: 1200 rows x ~6.7K
    nonzeros, secondary mode 2 sliced): every slice of every row counted
    once, lambda applied once, row sub-ranges (mttkrp_rows) included."""
    dims = (1200, 9000, 5000)
    idx, vals = synth.tensor(91, dims, 8_000_000, "uniform")
    npd = np.float64 if dtype == torch.float64 else np.float32
    vals = vals.astype(npd)
    A = factors_np(92, dims, R, npd)
    lam = np.linspace(0.5, 1.5, R).astype(npd)
    t = make(sp, dims, idx, vals, dtype)
    sp.build_perm(t, -1)
    A64 = [a.astype(np.float64) for a in A]
    Vo = oracle.mttkrp(dims, idx, vals.astype(np.float64), A64, 0, lam=lam.astype(np.float64))
    V = gpu_mttkrp(sp, t, 0, A, R, dtype, lam=lam)
    assert rel(V, Vo) <= TOL[dtype]
    A_dev = [dev(a, dtype) for a in A]
    out = torch.full((dims[0], R), float("nan"), dtype=dtype, device="cuda")
    sp.mttkrp_rows(t, 0, A_dev, out, 37, 1151, lam=dev(lam, dtype))
    got = out[37:1151].double().cpu().numpy()
    assert rel(got, Vo[37:1151]) <= TOL[dtype]


def test_max_size_mode_beyond_int32(sp):
    """A mode longer than 2^31 (32-bit keys: four radix passes; row offsets,
    rowptr searches and factor/out addresses past 2^32 elements need 64-bit
    arithmetic).  The oracle sees the same tensor with the long mode's used
    indices relabelled densely (MTTKRP is invariant under that relabelling)."""
    free, _ = torch.cuda.mem_get_info()
    if free < 100 * (1 << 30):
        pytest.skip("needs ~80 GB of free device memory")
    I0, R, P = (1 << 31) + 12345, 4, 60_000
    dims = (I0, 7, 5)
    rng = np.random.default_rng(7)
    used = np.unique(np.concatenate([rng.integers(0, I0, P // 3), [0, I0 - 1]]))
    idx = np.stack([rng.choice(used, P), rng.integers(0, 7, P), rng.integers(0, 5, P)], axis=1)
    vals = rng.random(P).astype(np.float32) + 0.5
    t = sp.sptensor_create(dims, dev(idx.astype(np.int64)), dev(vals))
    sp.build_perm(t, -1)
    p0, rp0 = gpu_perm(sp, t, 0)
    assert np.array_equal(p0, np.argsort(idx[:, 0], kind="stable").astype(np.uint32))
    assert int(rp0[-1]) == P and int(rp0[I0 - 1]) == P - int((idx[:, 0] == I0 - 1).sum())
    A0 = torch.rand(I0, R, dtype=torch.float32, device="cuda")
    A_d = [A0, dev(rng.random((7, R)).astype(np.float32)), dev(rng.random((5, R)).astype(np.float32))]
    # dense relabelling for the oracle
    rel_idx = idx.copy()
    rel_idx[:, 0] = np.searchsorted(used, idx[:, 0])
    A_h = [A0[torch.from_numpy(used).cuda()].double().cpu().numpy(),
           A_d[1].double().cpu().numpy(), A_d[2].double().cpu().numpy()]
    rdims = (len(used), 7, 5)
    for n in (1, 2):
        out = torch.empty((dims[n], R), dtype=torch.float32, device="cuda")
        sp.mttkrp(t, n, A_d, out)
        Vo = oracle.mttkrp(rdims, rel_idx, vals.astype(np.float64), A_h, n)
        assert rel(out.double().cpu().numpy(), Vo) <= TOL[torch.float32], n
    out0 = torch.empty((I0, R), dtype=torch.float32, device="cuda")
    sp.mttkrp(t, 0, A_d, out0)
    sample = np.array([0, 1, len(used) // 2, len(used) - 1])
    Vo = oracle.mttkrp_rows(rdims, rel_idx, vals.astype(np.float64), A_h, 0, sample)
    got = out0[torch.from_numpy(used[sample]).cuda()].double().cpu().numpy()
    assert rel(got, Vo) <= TOL[torch.float32]
    used_set = set(used[:64].tolist())
    empty = next(r for r in range(1, 64) if r not in used_set)
    assert float(out0[empty].abs().sum()) == 0.0                    # empty rows are exactly 0
    del out0, A0, A_d
    t.close()
    torch.cuda.empty_cache()


@pytest.mark.parametrize("layout", ["sorted", "perm_gather"])
def test_mttkrp_contention_and_empty_rows(sp, layout):
    """All nonzeros in one row (maximum contention), a 2-long mode, many empty rows."""
    dims = (5000, 2, 700)
    P = 300_000
    idx, vals = synth.tensor(5, dims, P, "uniform")
    idx[:, 0] = 4321
    A = factors_np(6, dims, 16)
    t = make(sp, dims, idx, vals, perm_gather=layout == "perm_gather")
    sp.build_perm(t, -1)
    for n in range(3):
        V = gpu_mttkrp(sp, t, n, A, 16, torch.float64)
        Vo = oracle.mttkrp(dims, idx, vals, A, n, acc_long=True)
        assert rel(V, Vo) <= 1e-12
        if n == 0:
            assert not np.delete(V, 4321, axis=0).any()          # exactly zero


def test_mttkrp_powerlaw_parity(sp):
    dims = (53200, 170000, 25000, 1400)
    P = 400_000
    idx, vals = synth.tensor(1813, dims, P, "powerlaw")
    A = factors_np(9179, dims, 16)
    t = make(sp, dims, idx, vals)
    sp.build_perm(t, -1)
    for n in range(4):
        V = gpu_mttkrp(sp, t, n, A, 16, torch.float64)
        Vo = oracle.mttkrp(dims, idx, vals, A, n, acc_long=True)
        assert rel(V, Vo) <= 1e-12


def test_host_buffers_and_errors(sp):
    dims = (10, 20, 30)
    idx, vals = synth.tensor(3, dims, 500)
    t = sp.sptensor_create(dims, idx.astype(np.int64), vals)          # numpy host buffers
    A = factors_np(4, dims, 8)
    with pytest.raises(sp.SptkError) as e:
        gpu_mttkrp(sp, t, 0, A, 8, torch.float64)
    assert e.value.name == "ENOPERM"
    sp.build_perm(t, -1)
    V = gpu_mttkrp(sp, t, 2, A, 8, torch.float64)
    assert rel(V, oracle.mttkrp(dims, idx, vals, A, 2)) <= 1e-12
    bad = idx.astype(np.int64).copy()
    bad[7, 1] = 20
    with pytest.raises(sp.SptkError) as e:
        sp.sptensor_create(dims, dev(bad), dev(vals))
    assert e.value.name == "ERANGE"
    bad[7, 1] = -1
    with pytest.raises(sp.SptkError) as e:
        sp.sptensor_create(dims, dev(bad), dev(vals))
    assert e.value.name == "ERANGE"
    with pytest.raises(sp.SptkError) as e:
        sp.build_perm(t, 3)
    assert e.value.name == "EINVAL"


# ------------------------------------------------------------------ synth
@pytest.mark.parametrize("source", ["pageable", "pinned", "mixed"])
def test_chunked_host_ingest(sp, source):
    """Host inputs are streamed in 1M-nonzero chunks (pinned staging, copy
    stream overlapped with the pack): a 9M-nonzero tensor (9 chunks, ragged
    last) built from pageable numpy, pinned torch, or host idx + device
    values gives the same records as the device-resident input -- bit-exact
    perms, equal MTTKRP, equal fit of one CP-ALS iteration."""
    dims = (3000, 2000, 1000)
    idx, vals = synth.tensor(97, dims, 9_000_000 + 123, "uniform")
    idx = idx.astype(np.int64)
    ref = sp.sptensor_create(dims, dev(idx), dev(vals))
    if source == "pageable":
        t = sp.sptensor_create(dims, idx, vals)
    elif source == "pinned":
        t = sp.sptensor_create(dims, torch.from_numpy(idx).pin_memory(),
                               torch.from_numpy(vals).pin_memory())
    else:
        t = sp.sptensor_create(dims, idx, dev(vals))
    for x in (ref, t):
        sp.build_perm(x, -1)
    A = [dev(a) for a in factors_np(98, dims, 8)]
    for n in range(3):
        assert np.array_equal(gpu_perm(sp, t, n)[0], gpu_perm(sp, ref, n)[0])
        o1 = torch.empty(dims[n], 8, dtype=torch.float64, device="cuda")
        o2 = torch.empty_like(o1)
        sp.mttkrp(t, n, A, o1)
        sp.mttkrp(ref, n, A, o2)
        assert rel(o1.cpu().numpy(), o2.cpu().numpy()) <= 1e-13
    F1 = [torch.empty(I, 8, dtype=torch.float64, device="cuda") for I in dims]
    F2 = [torch.empty(I, 8, dtype=torch.float64, device="cuda") for I in dims]
    r1 = sp.cp_als(t, 8, 1, F1, seed=5)
    r2 = sp.cp_als(ref, 8, 1, F2, seed=5)
    assert abs(r1["fit"] - r2["fit"]) <= 1e-9


def test_device_generator_matches_host():
    from synth import device
    for dist, dims in (("uniform", (12000, 9200, 28800)), ("powerlaw", (532000, 17_000_000, 1400))):
        idx_d, val_d = device.tensor(1812, dims, 100_000, dist, i0=12345)
        idx_h, val_h = synth.tensor(1812, dims, 100_000, dist, i0=12345)
        assert np.array_equal(idx_d.cpu().numpy().view(np.uint32), idx_h)
        assert np.array_equal(val_d.cpu().numpy(), val_h)
    f_d = device.factor(9178, 3, 1, 9200, 16)
    assert np.array_equal(f_d.cpu().numpy(), synth.factor(9178, 3, 1, 9200, 16))
    f32 = device.factor(9178, 3, 1, 100, 16, dtype=torch.float32)
    assert np.array_equal(f32.cpu().numpy(), synth.factor(9178, 3, 1, 100, 16, np.float32))


# ------------------------------------------------------------------ CP-ALS
def test_cp_als_tiny_trajectory(sp):
    c = synth.CONFIGS["tiny"]
    idx, vals = synth.unique_tensor(c.seed, c.dims, c.nnz)
    R = 8
    t = make(sp, c.dims, idx, vals)
    A = [torch.empty(I, R, dtype=torch.float64, device="cuda") for I in c.dims]
    lam = torch.empty(R, dtype=torch.float64, device="cuda")
    res = sp.cp_als(t, R, 10, A, tol=0.0, seed=c.seed_f, lambda_out=lam)
    ref = oracle.cp_als(c.dims, idx, vals, factors_np(c.seed_f, c.dims, R), 10)
    assert res["iters"] == ref["iters"] == 10
    assert np.max(np.abs(res["trace"] - ref["trace"])) <= 1e-9
    for m in range(3):
        assert rel(A[m].cpu().numpy(), ref["A"][m]) <= 1e-8
    assert rel(lam.cpu().numpy(), ref["lam"]) <= 1e-8
    # host factor buffers (end-to-end path): same result
    Ah = [np.empty((I, R)) for I in c.dims]
    lamh = np.empty(R)
    res2 = sp.cp_als(t, R, 10, Ah, seed=c.seed_f, lambda_out=lamh)
    # MTTKRP boundary rows use atomics (summation order varies run to run)
    assert np.max(np.abs(res2["trace"] - res["trace"])) <= 1e-12
    assert all(rel(Ah[m], A[m].cpu().numpy()) <= 1e-12 for m in range(3))
    assert rel(lamh, lam.cpu().numpy()) <= 1e-12
    # fp32: the oracle in fp64 on the fp32-rounded inputs; fit within 1e-4
    t32 = make(sp, c.dims, idx, vals.astype(np.float32), torch.float32)
    A32 = [torch.empty(I, R, dtype=torch.float32, device="cuda") for I in c.dims]
    res32 = sp.cp_als(t32, R, 10, A32, seed=c.seed_f)
    init32 = [a.astype(np.float32).astype(np.float64) for a in factors_np(c.seed_f, c.dims, R)]
    ref32 = oracle.cp_als(c.dims, idx, vals.astype(np.float32).astype(np.float64), init32, 10)
    assert np.max(np.abs(res32["trace"] - ref32["trace"])) <= 1e-4
    for m in range(3):
        assert rel(A32[m].double().cpu().numpy(), ref32["A"][m]) <= 1e-3


@pytest.mark.parametrize("deferred", [1, 0])
def test_cp_als_zero_column_ridge(sp, deferred):
    """Initial factors with a zero column make every Gamma singular (ridge
    retry) and that column of A_raw exactly zero (lambda_j = 0, column := e_1);
    the trajectory, factors and lambda still follow the oracle -- through the
    deferred-normalisation tail and the explicit one."""
    with sp.options(deferred_norm=deferred):
        _zero_column_ridge(sp)


def _zero_column_ridge(sp):
    c = synth.CONFIGS["tiny"]
    idx, vals = synth.unique_tensor(c.seed, c.dims, c.nnz)
    R = 6
    init = factors_np(c.seed_f, c.dims, R)
    for a in init:
        a[:, 2] = 0.0
    t = make(sp, c.dims, idx, vals)
    A = [dev(a) for a in init]
    lam = torch.empty(R, dtype=torch.float64, device="cuda")
    res = sp.cp_als(t, R, 6, A, init=[dev(a) for a in init], lambda_out=lam)
    ref = oracle.cp_als(c.dims, idx, vals, init, 6)
    assert np.max(np.abs(res["trace"] - ref["trace"])) <= 1e-9
    assert rel(lam.cpu().numpy(), ref["lam"]) <= 1e-8
    for m in range(3):
        assert rel(A[m].cpu().numpy(), ref["A"][m]) <= 1e-8
    # one iteration: mode 0's column 2 is exactly e_1 (lambda = 0 on the way)
    A1 = [dev(a) for a in init]
    sp.cp_als(t, R, 1, A1, init=[dev(a) for a in init])
    ref1 = oracle.cp_als(c.dims, idx, vals, init, 1)
    col = A1[0][:, 2].cpu().numpy()
    assert col[0] == 1.0 and not col[1:].any() and np.array_equal(col, ref1["A"][0][:, 2])


def test_cp_als_planted_recovery_and_f32(sp):
    dims = (400, 300, 500)
    idx, vals, mu, B = synth.planted_tensor(21, dims, 5, (60, 25, 20))
    t = make(sp, dims, idx, vals)
    A = [torch.empty(I, 5, dtype=torch.float64, device="cuda") for I in dims]
    res = sp.cp_als(t, 5, 60, A, seed=23)
    assert res["fit"] > 0.999
    ref = oracle.cp_als(dims, idx, vals, factors_np(23, dims, 5), 60)
    # near a perfect fit, fit = 1 - sqrt(res2)/||X|| with res2 a difference of
    # O(||X||^2) terms: |d fit| <= sqrt(c u) ~ 3e-8
    assert abs(res["fit"] - ref["fit"]) <= 1e-7
    t32 = make(sp, dims, idx, vals.astype(np.float32), torch.float32)
    A32 = [torch.empty(I, 5, dtype=torch.float32, device="cuda") for I in dims]
    res32 = sp.cp_als(t32, 5, 60, A32, seed=23)
    # same cancellation in fp32: |d fit| <= sqrt(c u32) ~ 5e-4
    assert res32["fit"] > 0.999 and abs(res32["fit"] - ref["fit"]) <= 1e-3


def test_cp_als_tol_and_errors(sp):
    dims = (400, 300, 500)
    idx, vals, mu, B = synth.planted_tensor(21, dims, 5, (60, 25, 20))
    t = make(sp, dims, idx, vals)
    A = [torch.empty(I, 5, dtype=torch.float64, device="cuda") for I in dims]
    res = sp.cp_als(t, 5, 200, A, tol=1e-6, seed=23)
    ref = oracle.cp_als(dims, idx, vals, factors_np(23, dims, 5), 200, tol=1e-6)
    assert res["iters"] == ref["iters"] < 200
    z = make(sp, (3, 3), np.array([[0, 0]]), np.array([0.0]))
    with pytest.raises(sp.SptkError) as e:
        sp.cp_als(z, 2, 3, [torch.empty(3, 2, dtype=torch.float64, device="cuda")] * 2)
    assert e.value.name == "EZERONORM"


# ------------------------------------------------------------------ full-size configs
def sampled_rows(counts, k=48, seed=0):
    rng = np.random.default_rng(seed)
    I = len(counts)
    rows = {0, I - 1, int(np.argmax(counts))}
    rows |= set(rng.choice(I, size=min(k, I), replace=False).tolist())
    return np.array(sorted(rows), dtype=np.int64)


U_ROUND = {torch.float64: 2.0 ** -53, torch.float32: 2.0 ** -24}


def row_errors(V, Vo):
    """Per-row relative Frobenius errors ||V_k - Vo_k|| / ||Vo_k|| (rows with
    Vo_k = 0 must be exactly 0: their error is ||V_k||)."""
    d = torch.linalg.vector_norm(V.double() - Vo, dim=1)
    nb = torch.linalg.vector_norm(Vo, dim=1)
    return torch.where(nb > 0, d / torch.where(nb > 0, nb, 1.0), d)


def row_tolerance(counts, N, dtype):
    """Per-row bound: the north-star normwise tolerance, widened
    for a row of n terms to 8 sqrt(n + N) u -- the statistical size of the
    rounding error of n positive terms summed in any order (each a product of
    N roundings) at 8 standard deviations; only rows far longer than the
    config's mean (power-law heads) reach it."""
    n = torch.as_tensor(counts, dtype=torch.float64, device="cuda")
    return torch.clamp(8.0 * torch.sqrt(n + N) * U_ROUND[dtype], min=TOL[dtype])


def full_config_check(sp, name, R, dtype, perm_gather=False):
    """Bench-sized input in the bench's launch configuration, compared on the
    FULL output: perms bit-exact (host counting sort), MTTKRP relative
    Frobenius over all rows <= TOL against oracle_mttkrp_omp (fp64, each row
    summed in storage order) and every row within row_tolerance."""
    from synth import device
    c = synth.CONFIGS[name]
    idx_d, val_d = device.tensor(c.seed, c.dims, c.nnz, c.dist, dtype=dtype)
    A_d = [device.factor(c.seed_f, c.N, m, I, R, dtype=dtype) for m, I in enumerate(c.dims)]
    t = sp.sptensor_create(c.dims, idx_d, val_d, perm_gather=perm_gather)
    sp.build_perm(t, -1)
    A_h = [a.double().cpu().numpy() for a in A_d]
    idx_h = idx_d.cpu().numpy().view(np.uint32)
    val_h = val_d.double().cpu().numpy()
    del idx_d, val_d
    worst = []
    for n in range(c.N):
        p, rp = gpu_perm(sp, t, n)
        po, rpo = oracle.perm(idx_h, n, c.dims[n])
        assert np.array_equal(p, po) and np.array_equal(rp, rpo), f"perm mode {n}"
        out = torch.empty((c.dims[n], R), dtype=dtype, device="cuda")
        sp.mttkrp(t, n, A_d, out)
        Vo = torch.from_numpy(oracle.mttkrp_omp(c.dims, idx_h, val_h, A_h, n, po, rpo)[0]).cuda()
        err = float(torch.linalg.vector_norm(out.double() - Vo) / torch.linalg.vector_norm(Vo))
        assert err <= TOL[dtype], f"mode {n}: rel-Fro {err:.3e} via {sp.last_dispatch()}"
        counts = np.diff(rpo.astype(np.int64))
        re = row_errors(out, Vo)
        tol = row_tolerance(counts, c.N, dtype)
        bad = re > tol
        assert not bool(bad.any()), (
            f"mode {n}: {int(bad.sum())} rows over their bound, worst row "
            f"{int(torch.argmax(re / tol))} err {float(re.max()):.3e}")
        worst.append((sp.last_dispatch(), err, float(re.max()), float((re / tol).max())))
    print(f"[{name} R{R} {dtype}] (dispatch, rel-Fro, worst row err, worst row err/bound): {worst}")
    return t


def test_config_lbnl_full(sp):
    full_config_check(sp, "lbnl", 16, torch.float64)


@pytest.mark.parametrize("R,dtype", [(16, torch.float64), (64, torch.float64),
                                     (16, torch.float32), (64, torch.float32)])
def test_config_nell2_full(sp, R, dtype):
    full_config_check(sp, "nell2", R, dtype)


def test_config_nell2_full_perm_gather(sp):
    full_config_check(sp, "nell2", 16, torch.float64, perm_gather=True)


@pytest.mark.parametrize("name,iters", [("lbnl", 3)])  # the oracle takes ~20 s here
def test_cp_als_full_size(sp, name, iters):
    """CP-ALS at BASELINE size against the oracle's trajectory: every glue
    path of the benchmarked iteration runs here -- the tensor-core apply over
    296 blocks on LBNL's 868K-row mode, the fused reduce + finalise, the
    small-mode last-block tails, the prioritised side-stream inverse, the
    filled slice grids, graph replay."""
    c = synth.CONFIGS[name]
    idx, vals = synth.tensor(c.seed, c.dims, c.nnz, c.dist)
    R = 16
    ref = oracle.cp_als(c.dims, idx, vals, factors_np(c.seed_f, c.dims, R), iters)
    t = make(sp, c.dims, idx, vals)
    F = [torch.empty(I, R, dtype=torch.float64, device="cuda") for I in c.dims]
    lam = torch.empty(R, dtype=torch.float64, device="cuda")
    res = sp.cp_als(t, R, iters, F, seed=c.seed_f, lambda_out=lam)
    assert np.max(np.abs(res["trace"] - ref["trace"])) <= 1e-9, (res["trace"], ref["trace"])
    assert rel(lam.cpu().numpy(), ref["lam"]) <= 1e-8
    for m in range(c.N):
        assert rel(F[m].cpu().numpy(), ref["A"][m]) <= 1e-8, m
    t.close()


def test_config_delicious_full(sp):
    full_config_check(sp, "delicious", 16, torch.float64)


@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("run", [4, 16, 256])
def test_mttkrp_worker_shapes(sp, variant, run):
    """Both worker shapes on the permuted copy (per-group runs / warp-
    cooperative steps) and several block lengths, incl. rows shorter and
    longer than a step, against the oracle."""
    dims = (300, 40, 7)
    idx, vals = synth.tensor(91, dims, 4 * 4096 + 77, "powerlaw")
    A = factors_np(92, dims, 16)
    t = make(sp, dims, idx, vals)
    sp.build_perm(t, -1)
    try:
        sp.set_tuning(variant, run)
        for n in range(3):
            V = gpu_mttkrp(sp, t, n, A, 16, torch.float64)
            assert rel(V, oracle.mttkrp(dims, idx, vals, A, n)) <= 1e-12, n
    finally:
        sp.set_tuning(-2, -2)


def test_device_generator_at_arbitrary_counters():
    from synth import device
    ids = np.array([0, 5, 1_699_999_999, 123456789, 77], dtype=np.uint32)
    ids_d = torch.from_numpy(ids.view(np.int32)).cuda()
    for dist, I in (("uniform", 4_800_000), ("powerlaw", 2_500_000)):
        got = device.coords_at(1814, 1, I, ids_d, dist).cpu().numpy().view(np.uint32)
        ref = np.array([synth.coords(1814, 1, I, int(i), 1, dist)[0] for i in ids])
        assert np.array_equal(got, ref)
    v = device.values_at(1814, 3, ids_d).cpu().numpy()
    assert np.array_equal(v, np.array([synth.values(1814, 3, int(i), 1)[0] for i in ids]))


def test_config_amazon_full(sp):
    """C5 at full size (1.7B nonzeros) in the bench's launch configuration.
    Host memory cannot hold the oracle's copy, so: the permutation is checked
    on the device against the generator (bijection, non-decreasing keys,
    increasing ids within ties, rowptr = key histogram), and the MTTKRP on
    sampled rows against oracle_mttkrp_rows on exactly those rows' nonzeros
    (selected through the verified perm/rowptr, coordinates and values
    regenerated from their counters)."""
    from synth import device
    import gc
    c = synth.CONFIGS["amazon"]
    R = 16
    gc.collect()                  # earlier tests' tensors and handles
    torch.cuda.empty_cache()
    free, total = torch.cuda.mem_get_info()
    if free < 170e9:
        pytest.skip(f"needs ~170 GB free device memory, have {free / 1e9:.0f} GB")
    idx_d, val_d = device.tensor(c.seed, c.dims, c.nnz, c.dist)
    t = sp.sptensor_create(c.dims, idx_d, val_d)
    del idx_d, val_d
    torch.cuda.empty_cache()
    sp.build_perm(t, -1)
    A_d = [device.factor(c.seed_f, c.N, m, I, R) for m, I in enumerate(c.dims)]
    A_h = [a.cpu().numpy() for a in A_d]
    P = c.nnz
    chunk = 200_000_000
    for n in range(c.N):
        out = torch.empty((c.dims[n], R), dtype=torch.float64, device="cuda")
        sp.mttkrp(t, n, A_d, out)
        V_rows = out  # kept until the sampled check
        perm = torch.empty(P, dtype=torch.int32, device="cuda")
        sp.get_perm(t, n, perm)
        rp = torch.empty(c.dims[n] + 1, dtype=torch.int32, device="cuda")
        sp.get_rowptr(t, n, rp)
        # bijection
        seen = torch.zeros(P, dtype=torch.bool, device="cuda")
        for s0 in range(0, P, chunk):
            seen[perm[s0:s0 + chunk].long()] = True
        assert bool(seen.all()), f"perm mode {n} is not a bijection"
        del seen
        counts = torch.zeros(c.dims[n], dtype=torch.int64, device="cuda")
        prev_key = prev_id = None
        for s0 in range(0, P, chunk):
            ids = perm[s0:s0 + chunk]
            keys = device.coords_at(c.seed, n, c.dims[n], ids, c.dist).long()
            idl = ids.long() & 0xFFFFFFFF
            if prev_key is not None:
                keys = torch.cat([prev_key, keys])
                idl = torch.cat([prev_id, idl])
            dk = keys[1:] - keys[:-1]
            assert bool((dk >= 0).all()), f"keys decrease in mode {n}"
            assert bool((idl[1:][dk == 0] > idl[:-1][dk == 0]).all()), f"unstable ties, mode {n}"
            counts += torch.bincount(keys[1:] if prev_key is not None else keys,
                                     minlength=c.dims[n])
            prev_key, prev_id = keys[-1:], idl[-1:]
        rph = rp.long()
        assert int(rph[0]) == 0 and int(rph[-1]) == P
        assert torch.equal(rph[1:] - rph[:-1], counts), f"rowptr mode {n}"
        # sampled rows
        rows = sampled_rows(counts.cpu().numpy(), k=24, seed=n)
        sel = torch.cat([perm[int(rph[r]):int(rph[r + 1])] for r in rows])
        sub_idx = np.stack([device.coords_at(c.seed, m, c.dims[m], sel, c.dist).cpu().numpy()
                            .view(np.uint32) for m in range(c.N)], axis=1)
        sub_val = device.values_at(c.seed, c.N, sel).cpu().numpy()
        Vo = oracle.mttkrp_rows(c.dims, sub_idx, sub_val, A_h, n, rows, acc_long=True)
        V = V_rows[torch.from_numpy(rows).cuda()].cpu().numpy()
        assert rel(V, Vo) <= 1e-12, f"mode {n}"
        del perm, V_rows, out
        torch.cuda.empty_cache()
    t.close()


@pytest.mark.parametrize("G", [2, 3, 8])
def test_simulated_row_shards(sp, G):
    """The multi-GPU work split on one device: each 'rank' computes its row
    range (sptk_partition_rows over rowptr_n) with sptk_mttkrp_rows into one
    buffer; the assembly equals the oracle (range edges use atomics)."""
    dims = (500, 9000, 64)
    idx, vals = synth.tensor(55, dims, 9 * 4096 + 3, "powerlaw")
    A = factors_np(56, dims, 16)
    t = make(sp, dims, idx, vals)
    sp.build_perm(t, -1)
    A_d = [dev(a) for a in A]
    for n in range(3):
        rp = gpu_perm(sp, t, n)[1]
        b = sp.partition_rows(rp, G)
        out = torch.full((dims[n], 16), float("nan"), dtype=torch.float64, device="cuda")
        for g in range(G):
            sp.mttkrp_rows(t, n, A_d, out, int(b[g]), int(b[g + 1]))
        torch.cuda.synchronize()
        assert rel(out.cpu().numpy(), oracle.mttkrp(dims, idx, vals, A, n)) <= 1e-12, n


@pytest.mark.parametrize("G,dims,P", [(2, (1200, 9000, 5000), 4_000_000),
                                      (3, (1200, 9000, 5000), 4_000_000),
                                      (2, (4800, 9000, 5000), 8_000_000)])   # slice path per shard
def test_shard_local_copies(sp, G, dims, P):
    """sptk_sptensor_set_shard: each rank's handle holds copies of its own row
    range only (smaller device footprint); its own rows match the oracle
    through the copy (per-group / cooperative / slice kernels, shifted copy
    base), and rows outside the shard still match (perm-gather)."""
    idx, vals = synth.tensor(95, dims, P, "uniform")
    A = factors_np(96, dims, 16)
    A_d = [dev(a) for a in A]
    full = make(sp, dims, idx, vals)
    sp.build_perm(full, -1)
    full_bytes = sp.sptensor_device_bytes(full)
    full.close()
    Vo = [oracle.mttkrp(dims, idx, vals, A, n) for n in range(3)]
    for g in range(G):
        t = make(sp, dims, idx, vals)
        sp.sptensor_set_shard(t, G, g)
        sp.build_perm(t, -1)
        assert sp.sptensor_device_bytes(t) < full_bytes
        for n in range(3):
            rp = gpu_perm(sp, t, n)[1]
            b = sp.partition_rows(rp, G)
            out = torch.full((dims[n], 16), float("nan"), dtype=torch.float64, device="cuda")
            sp.mttkrp_rows(t, n, A_d, out, int(b[g]), int(b[g + 1]))
            got = out[int(b[g]):int(b[g + 1])].cpu().numpy()
            assert rel(got, Vo[n][int(b[g]):int(b[g + 1])]) <= 1e-12, (g, n)
            other = (g + 1) % G   # rows of another shard: correct through perm_n
            out2 = torch.full((dims[n], 16), float("nan"), dtype=torch.float64, device="cuda")
            sp.mttkrp_rows(t, n, A_d, out2, int(b[other]), int(b[other + 1]))
            got2 = out2[int(b[other]):int(b[other + 1])].cpu().numpy()
            assert rel(got2, Vo[n][int(b[other]):int(b[other + 1])]) <= 1e-12, (g, n, "other")
        t.close()


@pytest.mark.parametrize("exchange", [0, 1, -1])
def test_sharded_code_path_one_rank(sp, monkeypatch, exchange):
    """The N>1 code path (partition, per-rank launches, NCCL all-reduce, the
    row exchange) driven through a real 1-rank NCCL communicator with
    SPTK_FORCE_SHARDED=1; results must match the oracle.  exchange = 0: rows
    replicated by grouped NCCL broadcasts; 1: the fused exchange, rows stored
    by the apply kernel through the symmetric window's peer mapping (here the
    rank's own copy seen through it); -1: the best the communicator supports
    (NVLS multimem where available)."""
    monkeypatch.setenv("SPTK_FORCE_SHARDED", "1")
    try:
        comm = sp.comm_create(sp.comm_unique_id(), 1, 0)
    except sp.SptkError as e:
        pytest.skip(f"NCCL unavailable: {e}")
    with sp.options(exchange=exchange):
        _sharded_one_rank(sp, comm, exchange)


def _sharded_one_rank(sp, comm, exchange):
    c = synth.CONFIGS["tiny"]
    idx, vals = synth.unique_tensor(c.seed, c.dims, c.nnz)
    R = 8
    t = make(sp, c.dims, idx, vals)
    sp.build_perm(t, -1)
    A = factors_np(c.seed_f, c.dims, R)
    A_d = [dev(a) for a in A]
    for n in range(3):
        out = torch.full((c.dims[n], R), float("nan"), dtype=torch.float64, device="cuda")
        sp.mttkrp(t, n, A_d, out, comm=comm)
        torch.cuda.synchronize()
        assert rel(out.cpu().numpy(), oracle.mttkrp(c.dims, idx, vals, A, n)) <= 1e-12
    F = [torch.empty(I, R, dtype=torch.float64, device="cuda") for I in c.dims]
    lam = torch.empty(R, dtype=torch.float64, device="cuda")
    res = sp.cp_als(t, R, 10, F, seed=c.seed_f, comm=comm, lambda_out=lam)
    ref = oracle.cp_als(c.dims, idx, vals, A, 10)
    assert np.max(np.abs(res["trace"] - ref["trace"])) <= 1e-9
    for m in range(3):
        assert rel(F[m].cpu().numpy(), ref["A"][m]) <= 1e-8
    assert rel(lam.cpu().numpy(), ref["lam"]) <= 1e-8
    mode = sp.comm_exchange(comm)
    print(f"exchange option {exchange}: agreed mode {mode}")
    if exchange >= 0:
        assert mode <= exchange
    # host factor buffers and a second call (the symmetric buffer is reused)
    Fh = [np.zeros((I, R)) for I in c.dims]
    res2 = sp.cp_als(t, R, 4, Fh, seed=c.seed_f, comm=comm)
    ref2 = oracle.cp_als(c.dims, idx, vals, A, 4)
    assert abs(res2["fit"] - ref2["fit"]) <= 1e-9
    for m in range(3):
        assert rel(Fh[m], ref2["A"][m]) <= 1e-8
    comm.close()


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
@pytest.mark.parametrize("dims,R,offset", [((57, 1203, 311), 16, 0), ((57, 1203, 311), 64, 0),
                                           ((40, 30, 20, 10), 17, 0), ((57, 1203, 311), 16, 1),
                                           ((500, 7), 300, 0)])
def test_mttkrp_atomic_variant(sp, dtype, dims, R, offset):
    """The paper's VerA/VerB traversal (storage order, atomics): no perm needed."""
    P = 3 * 4096 + 11
    idx, vals = synth.tensor(13, dims, P, "powerlaw")
    npd = np.float64 if dtype == torch.float64 else np.float32
    vals = vals.astype(npd)
    A = factors_np(14, dims, R, npd)
    lam = np.linspace(0.5, 1.5, R).astype(npd)
    t = make(sp, dims, idx, vals, dtype)
    for n in range(len(dims)):
        A_dev = []
        for a in A:
            buf = torch.zeros(a.size + offset, dtype=dtype, device="cuda")
            buf[offset:] = dev(a.reshape(-1), dtype)
            A_dev.append(buf[offset:].view(a.shape))
        out = torch.full((dims[n], R), float("nan"), dtype=dtype, device="cuda")
        sp.mttkrp_atomic(t, n, A_dev, out, lam=dev(lam, dtype))
        Vo = oracle.mttkrp(dims, idx, vals.astype(np.float64), [a.astype(np.float64) for a in A], n,
                           lam=lam.astype(np.float64))
        assert rel(out.double().cpu().numpy(), Vo) <= TOL[dtype], n


@pytest.mark.parametrize("R", [40, 100])
def test_cp_als_large_rank_tiled_glue(sp, R):
    """R > 32 takes the register-blocked glue (tiled V Gamma^{-1} and Gram)."""
    dims = (120, 130, 140)
    idx, vals = synth.unique_tensor(33, dims, 30000)
    t = make(sp, dims, idx, vals)
    F = [torch.empty(I, R, dtype=torch.float64, device="cuda") for I in dims]
    res = sp.cp_als(t, R, 6, F, seed=34)
    ref = oracle.cp_als(dims, idx, vals, factors_np(34, dims, R), 6)
    assert np.max(np.abs(res["trace"] - ref["trace"])) <= 1e-8
    for m in range(3):
        assert rel(F[m].cpu().numpy(), ref["A"][m]) <= 1e-6


@pytest.mark.parametrize("R,dtype,deferred", [
    (3, torch.float64, 1), (5, torch.float64, 1), (17, torch.float64, 1), (17, torch.float64, 0),
    (33, torch.float64, 1), (5, torch.float32, 1), (12, torch.float32, 1), (12, torch.float32, 0),
])
def test_cp_als_padded_rank(sp, R, dtype, deferred):
    """R not a multiple of the 32-byte lane vector: CP-ALS runs on factors
    padded with zero columns (DESIGN.md §4 "odd R").  The trajectory, the
    factors and lambda follow the oracle's rank-R run; pad_rank=0 (stride R,
    narrow lanes) gives the same result to rounding; device and host outputs
    agree."""
    dims = (150, 170, 130)
    idx, vals = synth.unique_tensor(41, dims, 20000)
    f32 = dtype == torch.float32
    v = vals.astype(np.float32).astype(np.float64) if f32 else vals
    init = factors_np(42, dims, R)
    if f32:
        init = [a.astype(np.float32).astype(np.float64) for a in init]
    ref = oracle.cp_als(dims, idx, v, init, 8)
    t = make(sp, dims, idx, vals.astype(np.float32) if f32 else vals, dtype)
    out = {}
    for pad in (1, 0):
        with sp.options(pad_rank=pad, deferred_norm=deferred):
            F = [torch.full((I, R), float("nan"), dtype=dtype, device="cuda") for I in dims]
            lam = torch.full((R,), float("nan"), dtype=dtype, device="cuda")
            res = sp.cp_als(t, R, 8, F, seed=42, lambda_out=lam)
            out[pad] = (res, [f.double().cpu().numpy() for f in F], lam.double().cpu().numpy())
    res, F, lam = out[1]
    tf, tl = (1e-4, 1e-3) if f32 else (1e-9, 1e-8)
    assert np.max(np.abs(res["trace"] - ref["trace"])) <= tf
    assert rel(lam, ref["lam"]) <= tl
    for m in range(3):
        assert rel(F[m], ref["A"][m]) <= tl, m
    res0, F0, lam0 = out[0]
    tp = 1e-4 if f32 else 1e-10
    assert np.max(np.abs(res0["trace"] - res["trace"])) <= tp
    for m in range(3):
        assert rel(F0[m], F[m]) <= (1e-3 if f32 else 1e-9)
    # host buffers (staged, strided copy-out) and the generator's init (no init)
    Fh = [np.full((I, R), np.nan, dtype=np.float32 if f32 else np.float64) for I in dims]
    resh = sp.cp_als(t, R, 8, Fh, seed=42)
    assert np.max(np.abs(resh["trace"] - res["trace"])) <= tp
    for m in range(3):
        assert rel(Fh[m], F[m]) <= (1e-3 if f32 else 1e-9)


@pytest.mark.parametrize("dims", [(90, 70), (60, 50, 40), (30, 25, 20, 15), (12, 11, 10, 9, 8)])
def test_cp_als_prezeroed_outputs(sp, dims):
    """The MTTKRP outputs zeroed on the side stream for the next mode (two
    buffers for even N, three for odd N; some zeroed in the same iteration,
    some in the previous one) give the oracle's trajectory, like zeroing in
    every launch (prezero=0), eagerly and through the replayed graph; also
    when the previous mode's apply launch zeroes it (zero_in_apply)."""
    P = min(int(np.prod(dims)) // 3, 4000)
    idx, vals = synth.unique_tensor(51, dims, P)
    R = 8
    ref = oracle.cp_als(dims, idx, vals, factors_np(52, dims, R), 7)
    t = make(sp, dims, idx, vals)
    for opts in ({"prezero": 2}, {"prezero": 0}, {"prezero": 2, "no_graph": 1},
                 {"prezero": 2, "zero_in_apply": 1}, {"prezero": 2, "zero_in_apply": 1, "no_graph": 1}):
        with sp.options(**opts):
            F = [torch.full((I, R), float("nan"), dtype=torch.float64, device="cuda") for I in dims]
            res = sp.cp_als(t, R, 7, F, seed=52)
            res2 = sp.cp_als(t, R, 7, F, seed=52)   # a second call replays the cached graph
        for r in (res, res2):
            assert np.max(np.abs(r["trace"] - ref["trace"])) <= 1e-9, opts
        for m in range(len(dims)):
            assert rel(F[m].cpu().numpy(), ref["A"][m]) <= 1e-8, (opts, m)


@pytest.mark.parametrize("R", [8, 16, 24, 32])
@pytest.mark.parametrize("inv", [{}, {"gj_warp": 0}, {"gamma_inv_chol": 1}])
def test_cp_als_inverse_kernels(sp, R, inv):
    """The one-warp Gauss-Jordan (default for R <= 32), the 256-thread one and
    the Cholesky inverse all follow the oracle's trajectory."""
    dims = (90, 80, 70)
    idx, vals = synth.unique_tensor(61, dims, 6000)
    ref = oracle.cp_als(dims, idx, vals, factors_np(62, dims, R), 6)
    t = make(sp, dims, idx, vals)
    with sp.options(**inv):
        F = [torch.empty(I, R, dtype=torch.float64, device="cuda") for I in dims]
        res = sp.cp_als(t, R, 6, F, seed=62)
    assert np.max(np.abs(res["trace"] - ref["trace"])) <= 1e-9
    for m in range(3):
        assert rel(F[m].cpu().numpy(), ref["A"][m]) <= 1e-7, m


@pytest.mark.parametrize("inv", [{}, {"gj_warp": 0}, {"gamma_inv_chol": 1}, {"deferred_norm": 0}])
def test_cp_als_duplicate_components(sp, inv):
    """Two identical CP components in the initial factors make every Gamma
    numerically singular (its pivot is rounding noise, often still positive):
    DESIGN.md §2 Z23 sends every inverse kernel to the ridge retry, like the
    oracle, so the trajectory stays finite, the fit rises monotonically (an
    ALS property), and it stays near the oracle's.  The split of the
    duplicate pair amplifies rounding by ~1/ridge = 1e12 (the oracle's pair
    grows to lambda ~ 2.4e3 against ~2 for the rest), so the trajectories
    drift apart (fits 0.0063 -> 0.0093; measured gaps 1e-5 after iteration 1,
    up to 4e-4 after 8 with the Cholesky kernel): the bar is finiteness,
    monotonicity, 5e-5 after the first iteration and 10 % after the last --
    not element parity."""
    dims = (90, 80, 70)
    R = 8
    idx, vals = synth.unique_tensor(63, dims, 6000)
    A0 = factors_np(64, dims, R)
    for a in A0:
        a[:, 1] = a[:, 0]
    ref = oracle.cp_als(dims, idx, vals, A0, 8)
    assert np.all(np.isfinite(ref["trace"]))
    t = make(sp, dims, idx, vals)
    with sp.options(**inv):
        F = [dev(a) for a in A0]
        lam = torch.empty(R, dtype=torch.float64, device="cuda")
        res = sp.cp_als(t, R, 8, F, init=F, lambda_out=lam)
    assert np.all(np.isfinite(res["trace"]))
    assert np.all(np.isfinite(lam.cpu().numpy()))
    tr = res["trace"]
    assert np.all(np.diff(tr) >= -1e-9), tr
    assert abs(tr[0] - ref["trace"][0]) <= 5e-5, (tr, ref["trace"])
    assert abs(tr[-1] - ref["trace"][-1]) <= 0.1 * ref["trace"][-1], (tr, ref["trace"])


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_window_major_copy(sp, dtype):
    """Window-major permuted copy (option win): a power-law 4-way tensor whose
    3rd mode has few rows and whose secondary factor spans many (shrunken)
    L2 windows.  The cooperative kernel reads rows from the records and
    red.adds every flush; MTTKRP of every mode and the CP-ALS trajectory
    follow the oracle, and a row sub-range call falls back to the perm
    gather."""
    dims = (3000, 200000, 40, 24)
    P = 600000
    idx, vals = synth.tensor(71, dims, P, "powerlaw")
    f32 = dtype == torch.float32
    v = vals.astype(np.float32).astype(np.float64) if f32 else vals
    R = 16
    A = factors_np(72, dims, R)
    if f32:
        A = [a.astype(np.float32).astype(np.float64) for a in A]
    with sp.options(win=1, slice_l2_kb=512):
        t = make(sp, dims, idx, vals.astype(np.float32) if f32 else vals, dtype)
        sp.build_perm(t, -1)
        for n in range(4):
            out = gpu_mttkrp(sp, t, n, A, R, dtype)
            kind = sp.last_dispatch()
            if n == 3 and not f32:  # fp32 N=4 records (16 B) have no spare row word
                assert "window" in kind, kind
            Vo = oracle.mttkrp(dims, idx, v, A, n)
            assert rel(out, Vo) <= TOL[dtype], (n, kind)
        # rows [5, 20) of mode 3: the window-major copy cannot serve a sub-range
        out = torch.full((dims[3], R), float("nan"), dtype=dtype, device="cuda")
        sp.mttkrp_rows(t, 3, [dev(a, dtype) for a in A], out, 5, 20)
        Vo = oracle.mttkrp(dims, idx, v, A, 3)
        assert rel(out[5:20].double().cpu().numpy(), Vo[5:20]) <= TOL[dtype]
        assert "window" not in sp.last_dispatch()
        if not f32:
            ref = oracle.cp_als(dims, idx, vals, factors_np(72, dims, R), 4)
            F = [torch.empty(I, R, dtype=dtype, device="cuda") for I in dims]
            res = sp.cp_als(t, R, 4, F, seed=72)
            assert np.max(np.abs(res["trace"] - ref["trace"])) <= 1e-9
        t.close()


def test_cp_als_degenerate_regime_reports_not_nan(sp):
    """CP-ALS deep into the degenerate regime of a random tensor (LBNL shape:
    columns collapse to lambda = 0 after ~50 iterations, Gamma can become
    numerically singular): every call either returns finite fits or raises
    SPTK_ESINGULAR -- never a silent NaN."""
    c = synth.CONFIGS["lbnl"]
    from synth import device
    idx, val = device.tensor(c.seed, c.dims, c.nnz, c.dist)
    t = sp.sptensor_create(c.dims, idx, val)
    sp.build_perm(t, -1)
    R = 16
    for its in (60, 90, 120):
        for prof in (False, True):
            F = [device.factor(c.seed_f, c.N, m, I, R) for m, I in enumerate(c.dims)]
            sp.profile_enable(prof)
            try:
                res = sp.cp_als(t, R, its, F, init=F)
                assert np.all(np.isfinite(res["trace"])), res["trace"]
                assert all(bool(torch.isfinite(f).all()) for f in F)
            except sp.SptkError as e:
                assert e.name == "ESINGULAR", e
            finally:
                sp.profile_enable(False)
    t.close()


@pytest.mark.parametrize("exchange", [0, 1])
def test_sharded_zero_column_e1(sp, monkeypatch, exchange):
    """A zero initial column through the sharded deferred path: every Gamma
    is singular (ridge retry), lambda_j = 0 and column j becomes e_1 on every
    replica -- the finalisation runs on each rank after the row exchange."""
    monkeypatch.setenv("SPTK_FORCE_SHARDED", "1")
    try:
        comm = sp.comm_create(sp.comm_unique_id(), 1, 0)
    except sp.SptkError as e:
        pytest.skip(f"NCCL unavailable: {e}")
    c = synth.CONFIGS["tiny"]
    idx, vals = synth.unique_tensor(c.seed, c.dims, c.nnz)
    R = 6
    init = factors_np(c.seed_f, c.dims, R)
    for a in init:
        a[:, 2] = 0.0
    t = make(sp, c.dims, idx, vals)
    with sp.options(exchange=exchange):
        A = [dev(a) for a in init]
        lam = torch.empty(R, dtype=torch.float64, device="cuda")
        res = sp.cp_als(t, R, 6, A, init=[dev(a) for a in init], lambda_out=lam, comm=comm)
        ref = oracle.cp_als(c.dims, idx, vals, init, 6)
        assert np.max(np.abs(res["trace"] - ref["trace"])) <= 1e-9
        assert rel(lam.cpu().numpy(), ref["lam"]) <= 1e-8
        for m in range(3):
            assert rel(A[m].cpu().numpy(), ref["A"][m]) <= 1e-8
        A1 = [dev(a) for a in init]
        sp.cp_als(t, R, 1, A1, init=[dev(a) for a in init], comm=comm)
        col = A1[0][:, 2].cpu().numpy()
        assert col[0] == 1.0 and not col[1:].any()
    comm.close()


def test_cp_als_large_rank_sharded_path(sp, monkeypatch):
    """R > 32 through the sharded (N>1) code path on one rank."""
    monkeypatch.setenv("SPTK_FORCE_SHARDED", "1")
    try:
        comm = sp.comm_create(sp.comm_unique_id(), 1, 0)
    except sp.SptkError as e:
        pytest.skip(f"NCCL unavailable: {e}")
    dims, R = (120, 130, 140), 40
    idx, vals = synth.unique_tensor(33, dims, 30000)
    t = make(sp, dims, idx, vals)
    F = [torch.empty(I, R, dtype=torch.float64, device="cuda") for I in dims]
    res = sp.cp_als(t, R, 6, F, seed=34, comm=comm)
    ref = oracle.cp_als(dims, idx, vals, factors_np(34, dims, R), 6)
    assert np.max(np.abs(res["trace"] - ref["trace"])) <= 1e-8
    for m in range(3):
        assert rel(F[m].cpu().numpy(), ref["A"][m]) <= 1e-6
    comm.close()


def test_mttkrp_property_random_shapes(sp):
    """Property sweep: random N in 1..6, dims (incl. length-1 and
    -2 modes), P in {0, 1, 2, ragged}, R in 1..70, dtype, distribution, layout
    -- every mode against the oracle."""
    hyp = pytest.importorskip("hypothesis")
    from hypothesis import given, settings, strategies as st

    @settings(max_examples=40, deadline=None, derandomize=True)
    @given(st.integers(1, 6), st.integers(0, 2**31 - 1), st.sampled_from([0, 1, 2, 37, 4096 + 5, 9000]),
           st.integers(1, 70), st.booleans(), st.booleans(), st.booleans())
    def run(N, seed, P, R, f32, powerlaw, pg):
        rng = np.random.default_rng(seed)
        dims = tuple(int(x) for x in rng.choice([1, 2, 3, 17, 64, 300, 5000], size=N))
        idx, vals = synth.tensor(seed % 10007, dims, P, "powerlaw" if powerlaw else "uniform")
        dtype = torch.float32 if f32 else torch.float64
        npd = np.float32 if f32 else np.float64
        vals = vals.astype(npd)
        A = factors_np(seed % 977, dims, R, npd)
        t = make(sp, dims, idx, vals, dtype, perm_gather=pg)
        sp.build_perm(t, -1)
        for n in range(N):
            V = gpu_mttkrp(sp, t, n, A, R, dtype)
            Vo = oracle.mttkrp(dims, idx, vals.astype(np.float64),
                               [a.astype(np.float64) for a in A], n)
            assert rel(V, Vo) <= TOL[dtype], (dims, P, R, n)

    run()


@pytest.mark.parametrize("variant,R", [(0, 16), (1, 16), (0, 10), (1, 6)])
@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_deterministic_mode_bitwise(sp, variant, R, dtype):
    """SPTK_CREATE_DETERMINISTIC: boundary rows summed in worker order ->
    repeated runs are bit-identical; values match the oracle; CP-ALS too."""
    dims = (3000, 200, 64)
    idx, vals = synth.tensor(61, dims, 40 * 4096 + 9, "powerlaw")   # hot rows span many workers
    npd = np.float64 if dtype == torch.float64 else np.float32
    vals = vals.astype(npd)
    A = factors_np(62, dims, R, npd)
    t = sp.sptensor_create(dims, dev(idx.astype(np.int64)), dev(vals, dtype), deterministic=True)
    sp.build_perm(t, -1)
    try:
        sp.set_tuning(variant, 16)
        for n in range(3):
            V1 = gpu_mttkrp(sp, t, n, A, R, dtype)
            V2 = gpu_mttkrp(sp, t, n, A, R, dtype)
            assert np.array_equal(V1, V2), n
            Vo = oracle.mttkrp(dims, idx, vals.astype(np.float64), [a.astype(np.float64) for a in A], n,
                               acc_long=True)
            assert rel(V1, Vo) <= TOL[dtype], n
    finally:
        sp.set_tuning(-2, -2)
    if dtype == torch.float64:
        F1 = [torch.empty(I, R, dtype=dtype, device="cuda") for I in dims]
        F2 = [torch.empty(I, R, dtype=dtype, device="cuda") for I in dims]
        r1 = sp.cp_als(t, R, 5, F1, seed=3)
        r2 = sp.cp_als(t, R, 5, F2, seed=3)
        assert np.array_equal(r1["trace"], r2["trace"])
        assert all(torch.equal(F1[m], F2[m]) for m in range(3))
    d2 = (300, 40)                                    # N = 2: generic kernel only
    i2, v2 = synth.tensor(63, d2, 999, "uniform")
    t2 = sp.sptensor_create(d2, dev(i2.astype(np.int64)), dev(v2.astype(npd), dtype),
                            deterministic=True)
    sp.build_perm(t2, -1)
    with pytest.raises(sp.SptkError) as e:
        gpu_mttkrp(sp, t2, 0, factors_np(64, d2, R, npd), R, dtype)
    assert e.value.name == "EUNSUPPORTED"


@pytest.mark.parametrize("variant", [0, 1])
def test_deterministic_rowrec_n4(sp, variant):
    """Deterministic mode on an N = 4 fp64 tensor, whose 32-byte copy records
    carry the row index (per-group kernel reads it from the record):
    repeated runs bit-identical, values match the oracle."""
    dims = (700, 90, 40, 2000)
    idx, vals = synth.tensor(65, dims, 30 * 4096 + 11, "powerlaw")
    R = 16
    A = factors_np(66, dims, R)
    t = sp.sptensor_create(dims, dev(idx.astype(np.int64)), dev(vals), deterministic=True)
    sp.build_perm(t, -1)
    try:
        sp.set_tuning(variant, 16)
        for n in range(4):
            V1 = gpu_mttkrp(sp, t, n, A, R, torch.float64)
            V2 = gpu_mttkrp(sp, t, n, A, R, torch.float64)
            assert np.array_equal(V1, V2), n
            Vo = oracle.mttkrp(dims, idx, vals, A, n, acc_long=True)
            assert rel(V1, Vo) <= 1e-12, n
    finally:
        sp.set_tuning(-2, -2)


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_duplicate_policies(sp, dtype):
    dims = (30, 20, 10)
    idx, vals = synth.tensor(19, dims, 20000)            # 6000 cells: many duplicates
    npd = np.float64 if dtype == torch.float64 else np.float32
    vals = vals.astype(npd)
    t = sp.sptensor_create(dims, dev(idx.astype(np.int64)), dev(vals, dtype), duplicates="sum")
    io, vo = oracle.merge_duplicates(idx, vals.astype(np.float64))
    assert t.nnz == len(io) == sptensor_nnz(sp, t)
    sp.build_perm(t, -1)
    A = factors_np(20, dims, 16, npd)
    for n in range(3):
        V = gpu_mttkrp(sp, t, n, A, 16, dtype)
        assert rel(V, oracle.mttkrp(dims, io, vo, [a.astype(np.float64) for a in A], n)) <= TOL[dtype]
        p, _ = gpu_perm(sp, t, n)
        assert np.array_equal(p, oracle.perm(io, n, dims[n])[0])   # merged storage order
    with pytest.raises(sp.SptkError) as e:
        sp.sptensor_create(dims, dev(idx.astype(np.int64)), dev(vals, dtype), duplicates="error")
    assert e.value.name == "EDUP"
    u, uv = synth.unique_tensor(21, dims, 500)
    tu = sp.sptensor_create(dims, dev(u.astype(np.int64)), dev(uv.astype(npd), dtype),
                            duplicates="error")
    assert tu.nnz == 500


def sptensor_nnz(sp, t):
    return sp.sptensor_info(t)["nnz"]


def test_c_api_demo(sp, tmp_path):
    """The C ABI from plain C (examples/c_api_demo.c): build with gcc, run."""
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = tmp_path / "c_api_demo"
    libdir = os.path.join(root, "paper_1809_09175_b200")
    subprocess.check_call(["gcc", "-O2", "-I", os.path.join(root, "include"),
                           "-I", "/usr/local/cuda/include", os.path.join(root, "examples", "c_api_demo.c"),
                           "-L", libdir, "-l:libsptk.so", "-L", "/usr/local/cuda/lib64", "-lcudart",
                           f"-Wl,-rpath,{libdir}:/usr/local/cuda/lib64", "-lm", "-o", str(exe)])
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "c_api_demo ok" in r.stdout
