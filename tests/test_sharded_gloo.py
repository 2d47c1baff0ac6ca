"""Multi-process (world_size 2, gloo, CPU) test of the N>1 decomposition the
library uses: rows of mode n are split with the library's own
host partitioner (sptk_partition_rows), each rank computes only its rows --
MTTKRP and the ALS row solve -- the R column sums of squares are all-reduced
and the row blocks all-gathered.  Per-rank math is the oracle's; the
assembled result must equal the single-process oracle."""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _worker(rank, world, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import oracle
        import paper_1809_09175_b200 as sp
        import synth
        dims = (300, 250, 40)
        idx, vals = synth.tensor(77, dims, 20000, "powerlaw")
        R = 6
        A = [synth.factor(78, 3, m, I, R) for m, I in enumerate(dims)]
        ok = []
        newA = [a.copy() for a in A]
        G = [a.T @ a for a in A]
        for n in range(3):
            perm, rowptr = oracle.perm(idx, n, dims[n])
            b = sp.partition_rows(rowptr, world)                 # library host logic
            r0, r1 = int(b[rank]), int(b[rank + 1])
            mine = perm[rowptr[r0]:rowptr[r1]]                    # this rank's positions
            V = oracle.mttkrp_rows(dims, idx[mine], vals[mine], newA, n, np.arange(r0, r1))
            # gather row blocks (padded) and assemble
            maxr = int(np.max(np.diff(b)))
            pad = np.zeros((maxr, R))
            pad[: r1 - r0] = V
            parts = [torch.zeros(maxr, R, dtype=torch.float64) for _ in range(world)]
            dist.all_gather(parts, torch.from_numpy(pad))
            full = np.concatenate([parts[g].numpy()[: b[g + 1] - b[g]] for g in range(world)])
            ok.append(np.allclose(full, oracle.mttkrp(dims, idx, vals, newA, n), rtol=1e-13, atol=0))
            # ALS row update on own rows; column norms all-reduced
            Gam = np.ones((R, R))
            for m in range(3):
                if m != n:
                    Gam *= G[m]
            An = oracle.chol_solve(Gam, V) if r1 > r0 else np.zeros((0, R))
            colsq = torch.from_numpy((An ** 2).sum(axis=0))
            dist.all_reduce(colsq)
            lam = np.sqrt(colsq.numpy())
            pad = np.zeros((maxr, R))
            pad[: r1 - r0] = An / lam
            dist.all_gather(parts, torch.from_numpy(pad))
            newA[n] = np.concatenate([parts[g].numpy()[: b[g + 1] - b[g]] for g in range(world)])
            G[n] = newA[n].T @ newA[n]
        ref = oracle.cp_als(dims, idx, vals, A, 1)
        ok.append(all(np.allclose(newA[m], ref["A"][m], rtol=1e-9, atol=1e-12) for m in range(3)))
        ok.append(np.allclose(lam, ref["lam"], rtol=1e-9))
        q.put((rank, ok))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))


def test_two_rank_row_sharding_matches_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, ok in res:
        assert isinstance(ok, list), ok
        assert all(ok), (rank, ok)
