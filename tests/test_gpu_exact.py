"""Integer-exact MTTKRP parity at full size, through every traversal.

Pin (DESIGN.md §5 "integer-exact pins"): with integer values x in {1..4} and
integer factor entries in {1..3} (synth.int_values / synth.int_factor: the
same draws as the regular inputs mapped to small integers), every term
x_i * prod_{m != n} A_m(l_im, j) of Eq. (2) is an integer and every
partial sum stays below 2^53 (fp64) / 2^24 (fp32), so any summation order --
atomics, slices, warp shuffles, worker partials -- gives the exact result.
The GPU output must therefore equal the oracle's BIT FOR BIT: a dropped,
duplicated or misrouted nonzero, a wrong gathered row or a lost atomic changes
an integer and fails.

Every BASELINE config (C1-C5) at its full size, every traversal the library
has (forced in-process with sp.options; sp.last_dispatch() proves which kernel
ran):  the default choice, the slice traversal (forced, and in its L2-window
regime), the warp-cooperative and per-group kernels (with and without the row
index in the record), narrow lane vectors (V = 1: column tiles for R = 64),
the generic scalar kernel, the paper's perm-gather traversal, the
atomic-per-nonzero traversal (VerA/VerB), deterministic mode and row-range
shards (sptk_mttkrp_rows over sptk_partition_rows).  A second, oracle-free
pin: with all factors = 1 the output row k is sum_{i in row k} x_i in every
column, i.e. numpy's bincount of the mode-n coordinates weighted by x.
"""
import gc

import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

CASES = [("tiny", 8, "f64"), ("lbnl", 16, "f64"), ("nell2", 16, "f64"), ("nell2", 64, "f64"),
         ("nell2", 16, "f32"), ("nell2", 64, "f32"), ("delicious", 16, "f64"),
         ("amazon", 16, "f64")]
TDT = {"f64": torch.float64, "f32": torch.float32}
EXACT_LIMIT = {"f64": 2.0 ** 53, "f32": 2.0 ** 24}

# name -> (options, expected dispatch tag, applies(case) predicate)
TRAVERSALS = {
    "default": ({}, "", None),
    "slice": ({"slice": 2}, "slice", None),
    "slice_l2window": ({"slice": 2, "slice_l2_kb": 64}, "slice_l2window", None),
    "coop": ({"slice": 0, "variant": 1}, "coop", None),
    "fast": ({"slice": 0, "variant": 0, "rowrec": 0}, "fast V", None),
    "fast_rowrec": ({"slice": 0, "variant": 0, "rowrec": 1}, "fast_rowrec",
                    lambda c, dt: (dt == "f64" and c.N >= 4) or (dt == "f32" and c.N == 5)),
    "narrow_v1": ({"force_v": 1}, " V1", None),
    "generic": ({"generic": 1}, "generic", None),
    "perm_gather": ({"use_copy": 0}, "perm_gather", None),
    "atomic": ({}, "atomic", None),
    "rows_g3": ({}, "", None),
    "deterministic": ({}, "+det", None),
}


@pytest.fixture(scope="module")
def sp():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import paper_1809_09175_b200 as sp
    sp.lib()
    return sp


class Case:
    """One config with integer inputs: device tensor handle + oracle outputs."""

    def __init__(self, sp, name, R, dt):
        from synth import device
        c = synth.CONFIGS[name]
        self.c, self.R, self.dt, self.tdt = c, R, dt, TDT[dt]
        gc.collect()
        torch.cuda.empty_cache()
        if name == "amazon":
            free, _ = torch.cuda.mem_get_info()
            if free < 170e9:
                pytest.skip(f"needs ~170 GB free device memory, have {free / 1e9:.0f} GB")
        idx_d, val_d = device.tensor(c.seed, c.dims, c.nnz, c.dist)
        vint_d = device.int_values_from(val_d)
        del val_d
        self.idx = idx_d.cpu().numpy().view(np.uint32)
        self.vals = vint_d.cpu().numpy()
        self.vals_dev = vint_d.to(self.tdt)
        del vint_d
        if name == "amazon":   # ingest from host (chunked): keeps device memory for the copies
            del idx_d
            self.vals_dev = None
            torch.cuda.empty_cache()
            self.t = sp.sptensor_create(c.dims, self.idx.view(np.int32),
                                        self.vals.astype(np.float64))
        else:
            self.t = sp.sptensor_create(c.dims, idx_d, self.vals_dev)
            self.idx_dev = idx_d
        sp.build_perm(self.t, -1)
        self.A = [synth.int_factor(c.seed_f, c.N, m, I, R) for m, I in enumerate(c.dims)]
        self.A_dev = [device.int_factor(c.seed_f, c.N, m, I, R, dtype=self.tdt)
                      for m, I in enumerate(c.dims)]
        for a, ad in zip(self.A, self.A_dev):   # host and device integers agree
            assert torch.equal(torch.from_numpy(a).to(self.tdt).cuda(), ad)
        self.perm = []
        self.V = []
        for n in range(c.N):
            po, rpo = oracle.perm(self.idx, n, c.dims[n])
            Vo, _ = oracle.mttkrp_omp(c.dims, self.idx, self.vals, self.A, n, po, rpo)
            assert float(Vo.max(initial=0.0)) < EXACT_LIMIT[dt], "integer sums must stay exact"
            self.perm.append((po, rpo))
            self.V.append(torch.from_numpy(Vo).to(self.tdt).cuda())

    def close(self):
        self.t.close()


@pytest.fixture(scope="module", params=CASES, ids=[f"{n}-R{r}-{d}" for n, r, d in CASES])
def case(sp, request):
    k = Case(sp, *request.param)
    yield k
    k.close()
    del k
    gc.collect()
    torch.cuda.empty_cache()


def _run(sp, k, n, trav):
    """Output of mode n through traversal `trav` (fresh NaN-filled buffer)."""
    out = torch.full((k.c.dims[n], k.R), float("nan"), dtype=k.tdt, device="cuda")
    if trav == "atomic":
        sp.mttkrp_atomic(k.t, n, k.A_dev, out)
    elif trav == "rows_g3":
        b = sp.partition_rows(k.perm[n][1], 3)
        for g in range(3):
            sp.mttkrp_rows(k.t, n, k.A_dev, out, int(b[g]), int(b[g + 1]))
    else:
        sp.mttkrp(k.t, n, k.A_dev, out)
    torch.cuda.synchronize()
    return out


@pytest.mark.parametrize("trav", list(TRAVERSALS))
def test_integer_exact_every_traversal(sp, case, trav):
    k = case
    opts, tag, applies = TRAVERSALS[trav]
    if applies is not None and not applies(k.c, k.dt):
        pytest.skip(f"{trav}: no such kernel for N={k.c.N} {k.dt}")
    t_det = None
    if trav == "deterministic":
        if k.c.name == "amazon":
            pytest.skip("deterministic mode needs a second 1.7B-nonzero handle")
        t_det = sp.sptensor_create(k.c.dims, k.idx_dev, k.vals_dev, deterministic=True)
        sp.build_perm(t_det, -1)
    seen = []
    try:
        with sp.options(**opts):
            for n in range(k.c.N):
                if t_det is not None:
                    out = torch.full((k.c.dims[n], k.R), float("nan"), dtype=k.tdt, device="cuda")
                    sp.mttkrp(t_det, n, k.A_dev, out)
                    torch.cuda.synchronize()
                else:
                    out = _run(sp, k, n, trav)
                d = sp.last_dispatch()
                seen.append(d)
                assert torch.equal(out, k.V[n]), (
                    f"mode {n} via {d}: {int((out != k.V[n]).sum())} entries differ, "
                    f"max |diff| {float((out.double() - k.V[n].double()).abs().nan_to_num(1e300).max())}")
    finally:
        if t_det is not None:
            t_det.close()
    print(f"[{k.c.name} R{k.R} {k.dt}] {trav}: {seen}")
    if tag and not any(tag in d for d in seen):
        pytest.skip(f"{trav} not reachable on this shape (ran {seen})")


def test_rowsum_bincount_pin(sp, case):
    """Oracle-free pin: all factors = 1 -> V(k, :) = sum of x over row k
    (numpy bincount of the coordinates, weighted by the integer values)."""
    k = case
    ones = [torch.ones((I, k.R), dtype=k.tdt, device="cuda") for I in k.c.dims]
    for n in range(k.c.N):
        out = torch.full((k.c.dims[n], k.R), float("nan"), dtype=k.tdt, device="cuda")
        sp.mttkrp(k.t, n, ones, out)
        torch.cuda.synchronize()
        rs = np.bincount(k.idx[:, n], weights=k.vals, minlength=k.c.dims[n])
        exp = torch.from_numpy(rs).to(k.tdt).cuda()[:, None].expand(-1, k.R)
        assert torch.equal(out, exp), f"mode {n} via {sp.last_dispatch()}"
