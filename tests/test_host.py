"""CPU-only tests of the product's host side: the C-ABI library loads and
exports every symbol include/sptk.h declares, host-only logic (row
partitioning, argument validation that fails before any CUDA call), the byte
models, and the input generator's determinism."""
import json
import os
import re

import numpy as np
import pytest

import synth
from paper_1809_09175_b200 import metrics

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = json.load(open(os.path.join(ROOT, "tests", "golden", "spec_examples.json")))


@pytest.fixture(scope="module")
def sp():
    import paper_1809_09175_b200 as sp
    from paper_1809_09175_b200 import build
    build.build()
    sp.lib()
    return sp


def test_library_exports_every_header_symbol(sp):
    header = open(os.path.join(ROOT, "include", "sptk.h")).read()
    header = re.sub(r"/\*.*?\*/", "", header, flags=re.S)          # drop comments
    declared = set(re.findall(r"\b(sptk_[a-z_0-9]+)\s*\(", header))
    assert len(declared) >= 18
    lib = sp.lib()
    for name in declared:
        assert hasattr(lib, name), name
    assert set(sp.EXPORTS) == declared
    assert "sm_100a" in sp.version()


def test_partition_rows_definition(sp):
    rng = np.random.default_rng(0)
    for In, nr in [(1, 1), (1, 4), (10, 3), (1000, 8), (50, 2)]:
        counts = rng.integers(0, 20, In)
        if In > 3:
            counts[3] = 500          # one hot row
        rowptr = np.concatenate([[0], np.cumsum(counts)]).astype(np.uint32)
        b = sp.partition_rows(rowptr, nr)
        P = int(rowptr[-1])
        assert b[0] == 0 and b[-1] == In and np.all(np.diff(b) >= 0)
        for g in range(1, nr):
            target = -(-P * g // nr)
            expect = int(np.searchsorted(rowptr, target, side="left"))
            assert b[g] == min(expect, In)


def test_create_validation_before_cuda(sp):
    with pytest.raises(sp.SptkError) as e:
        sp.sptensor_create([], np.zeros((0, 0), np.int64), np.zeros(0))
    assert e.value.name == "EUNSUPPORTED"
    with pytest.raises(sp.SptkError) as e:
        sp.sptensor_create([3, 0], np.zeros((1, 2), np.int64), np.zeros(1))
    assert e.value.name == "EUNSUPPORTED"
    with pytest.raises(sp.SptkError) as e:
        sp.sptensor_create([2] * 7, np.zeros((1, 7), np.int64), np.zeros(1))
    assert e.value.name == "EUNSUPPORTED"
    with pytest.raises(ValueError):
        sp.sptensor_create([2, 2], np.zeros((3, 2), np.int64), np.zeros(2))


def test_metrics_golden():
    for key in ("storage_base", "storage_small"):
        g = GOLD[key]
        assert metrics.storage_bytes(g["d"], g["P"], g["s_r"], g["s_o"], False) == g["base"], g["cite"]
        assert metrics.storage_bytes(g["d"], g["P"], g["s_r"], g["s_o"], True) == g["with_perm"], g["cite"]
    g = GOLD["bandwidth_model"]
    assert metrics.paper_bandwidth(g["d"], g["R"], g["P"], g["s_r"], g["s_o"], g["t"]) == pytest.approx(
        g["bytes_per_s"], rel=1e-12), g["cite"]
    for d, R, f in GOLD["flops_spec"]["cases"]:
        assert metrics.flops_spec(d, R) == f
    # C3 f64 R=16 B_model = 21.3 GB per mode (avg over modes)
    c = synth.CONFIGS["nell2"]
    bm = np.mean([metrics.b_model(3, c.nnz, 16, I, 8) for I in c.dims])
    assert bm == pytest.approx(21.3e9, rel=0.01)


def test_synth_deterministic_and_ranges():
    a = synth.tensor(5, (7, 9, 1), 1000, "uniform")
    b = synth.tensor(5, (7, 9, 1), 1000, "uniform")
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    assert a[0][:, 0].max() == 6 and a[0][:, 2].max() == 0
    assert (a[1] > 0).all() and (a[1] <= 1).all()
    # the chunked generation is the same stream
    c = synth.tensor(5, (7, 9, 1), 600, "uniform", i0=400)
    assert np.array_equal(c[0], a[0][400:])
    p = synth.tensor(6, (1400, 2), 20000, "powerlaw")[0][:, 0]
    top = np.bincount(p).max() / len(p)
    assert abs(top - np.log(2) / np.log(1401)) < 0.01    # Zipf(1) head mass
    f = synth.factor(3, 3, 1, 5, 4)
    assert f.shape == (5, 4) and (f >= 0).all() and (f < 1).all()


def test_bench_reference_arm_contract():
    """bench.py --impl reference (the oracle arm, CPU only) prints one JSON
    line with the driver's keys; run on the tiny config."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference",
                        "--config", "tiny", "--steps", "2", "--warmup", "1"],
                       capture_output=True, text=True, timeout=600, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "impl", "cpu_baseline", "e2e", "config", "dtype"):
        assert k in line, k
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["steps"] == 2


def test_options_roundtrip_and_unknown_name(sp):
    """Launch options (include/sptk.h): set/get/restore in-process, unknown
    names are SPTK_EINVAL, the context manager restores the previous value."""
    assert sp.get_option("slice") == 1
    with sp.options(slice=0, slice_l2_kb=3):
        assert sp.get_option("slice") == 0 and sp.get_option("slice_l2_kb") == 3
    assert sp.get_option("slice") == 1 and sp.get_option("slice_l2_kb") == 32768
    with pytest.raises(sp.SptkError) as e:
        sp.set_option("no_such_option", 1)
    assert e.value.name == "EINVAL"
    sp.set_tuning(1, 64)
    assert sp.get_option("variant") == 1 and sp.get_option("run") == 64
    sp.reset_options()
    assert sp.get_option("variant") == -1 and sp.get_option("run") == 0
    assert sp.last_dispatch() == ""


def test_every_documented_option_exists_with_its_default(sp):
    """Every option include/sptk.h documents is known to the library, with the
    documented default (round-2 options included)."""
    import re
    hdr = open(os.path.join(ROOT, "include", "sptk.h")).read()
    doc = hdr[hdr.index("sptk_set_option") - 7000:hdr.index("sptk_status sptk_set_option")]
    defaults = {"pad_rank": 1, "sort_v1": 0, "prezero": 1, "apply_mma": 1, "gj_warp": 1,
                "side_prio": -1, "win": 0, "slice_fill": 6, "fused_reduce": 1, "prezero_mb": 256, "zero_in_apply": 0, "exchange": -1,
                "pdl": 1, "keep_keys": 1, "tail_rows": 8192, "slice": 1, "slice_l2_kb": 32768}
    sp.reset_options()
    for name, value in defaults.items():
        assert sp.get_option(name) == value, name
    for name in re.findall(r"\b([a-z][a-z0-9_]+) -?[0-9]+ \(", doc):
        sp.get_option(name)  # raises SptkError if the library does not know it


def test_binding_validates_buffers_before_the_abi(sp):
    """shapes, dtypes, contiguity and placement are checked in the
    binding before raw addresses cross the C ABI (a float32 factor for an f64
    tensor, a short factor, a host buffer where a device pointer is required,
    or a wrong-dtype host buffer for cp_als's device-to-host copies)."""
    t = sp.SpTensor(0, (4, 5, 6), 10, sp.F64)
    ok = [np.zeros((I, 3)) for I in (4, 5, 6)]
    out = np.zeros((5, 3))
    # mttkrp takes device pointers only: host numpy is refused up front
    with pytest.raises(ValueError, match="CUDA tensor"):
        sp.mttkrp(t, 1, ok, out)
    with pytest.raises(ValueError, match="shape"):
        sp.mttkrp(t, 1, ok, np.zeros((4, 3)))
    with pytest.raises(ValueError, match="mode"):
        sp.mttkrp(t, 3, ok, out)
    with pytest.raises(ValueError, match="matrices"):
        sp.mttkrp_rows(t, 0, ok[:2], np.zeros((4, 3)), 0, 4)
    # cp_als accepts host buffers, but each must be (I_m, R) of the dtype
    with pytest.raises(ValueError, match="dtype"):
        sp.cp_als(t, 3, 1, [a.astype(np.float32) for a in ok])
    with pytest.raises(ValueError, match="shape"):
        sp.cp_als(t, 3, 1, [ok[0], ok[1], np.zeros((5, 3))])
    with pytest.raises(ValueError, match="contiguous"):
        sp.cp_als(t, 3, 1, [ok[0], ok[1], np.zeros((3, 6)).T])
    with pytest.raises(ValueError, match="lambda_out"):
        sp.cp_als(t, 3, 1, ok, lambda_out=np.zeros(4))
    with pytest.raises(ValueError, match="init"):
        sp.cp_als(t, 3, 1, ok, init=[ok[0], ok[1], np.zeros((6, 2))])
    t.handle = None  # never a real handle: nothing to destroy
