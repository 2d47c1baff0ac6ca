"""Multi-rank NCCL parity (needs >= 2 GPUs; skipped otherwise): libsptk's
sharded MTTKRP and CP-ALS over a real 2-rank communicator -- per-rank row
ranges with shard-local copies, the fused row exchange (NVLS multimem or
NVLink peer stores from the apply kernel) and the NCCL-broadcast fallback,
the all-reduced column norms / Gram matrices / fit, the e_1 rule for a zero
column on the rank that owns row 0 -- against the single-process oracle
(ADVICE r1)."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("exchange", [-1, 1, 0])
def test_two_rank_sharded_parity(tmp_path, exchange):
    if torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs (this box has %d)" % torch.cuda.device_count())
    out = tmp_path / "r0.npz"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "tests", "_multirank_worker.py"), str(out), str(exchange)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    got = np.load(out)
    dims, R = (300, 257, 190), 8
    idx, vals = synth.unique_tensor(77, dims, 20000)
    A = [synth.factor(78, 3, m, I, R) for m, I in enumerate(dims)]
    for n in range(3):
        Vo = oracle.mttkrp(dims, idx, vals, A, n)
        assert np.linalg.norm(got[f"V{n}"] - Vo) / np.linalg.norm(Vo) <= 1e-12, n
    ref = oracle.cp_als(dims, idx, vals, [synth.factor(79, 3, m, I, R) for m, I in enumerate(dims)], 10)
    assert np.max(np.abs(got["trace"] - ref["trace"])) <= 1e-9
    for m in range(3):
        assert np.linalg.norm(got[f"F{m}"] - ref["A"][m]) / np.linalg.norm(ref["A"][m]) <= 1e-8
    assert np.linalg.norm(got["lam"] - ref["lam"]) / np.linalg.norm(ref["lam"]) <= 1e-8
    if exchange >= 0:
        assert int(got["mode"]) <= exchange
