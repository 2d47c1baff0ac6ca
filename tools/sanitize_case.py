"""Small end-to-end case for compute-sanitizer (one tool per run): create,
build_perm, every MTTKRP path (permuted copy per-group / warp-cooperative,
perm-gather, generic, atomic, row shards) and CP-ALS (R=8 and R=40)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1809_09175_b200 as sp  # noqa: E402
import synth  # noqa: E402

dims = (300, 40, 7)
idx, vals = synth.tensor(91, dims, 3 * 4096 + 77, "powerlaw")
for pg in (False, True):
    t = sp.sptensor_create(dims, torch.from_numpy(idx.astype(np.int64)).cuda(),
                           torch.from_numpy(vals).cuda(), perm_gather=pg)
    sp.build_perm(t, -1)
    for R in (8, 16, 17, 40):
        A = [torch.rand(I, R, dtype=torch.float64, device="cuda") for I in dims]
        for n in range(3):
            out = torch.empty(dims[n], R, dtype=torch.float64, device="cuda")
            for v in (0, 1):
                sp.set_tuning(v, 0)
                sp.mttkrp(t, n, A, out)
            sp.set_tuning(-2, -2)
            sp.mttkrp_atomic(t, n, A, out)
            sp.mttkrp_rows(t, n, A, out, 0, dims[n] // 2)
            sp.mttkrp_rows(t, n, A, out, dims[n] // 2, dims[n])
    for R in (8, 40):
        F = [torch.empty(I, R, dtype=torch.float64, device="cuda") for I in dims]
        sp.cp_als(t, R, 5, F, seed=1)
    torch.cuda.synchronize()
print("sanitize case done")

# later paths: slice traversal (L1 windows), row index in 32-byte copy records
# (N = 4 fp64), chunked host ingest (2 chunks), shard-local copies, deterministic
dims = (2400, 4096, 3000)
idx, vals = synth.tensor(93, dims, 200_000, "uniform")
t = sp.sptensor_create(dims, idx.astype(np.int64), vals)          # host ingest path
sp.build_perm(t, -1)
A = [torch.rand(I, 16, dtype=torch.float64, device="cuda") for I in dims]
for n in range(3):
    out = torch.empty(dims[n], 16, dtype=torch.float64, device="cuda")
    sp.mttkrp(t, n, A, out)
    sp.mttkrp_rows(t, n, A, out, 100, dims[n] - 100)
t.close()
big = synth.tensor(94, (300, 200, 100), 1_100_000, "uniform")       # > 1 ingest chunk
t = sp.sptensor_create((300, 200, 100), big[0].astype(np.int64), big[1])
sp.sptensor_set_shard(t, 2, 1)
sp.build_perm(t, -1)
A = [torch.rand(I, 8, dtype=torch.float64, device="cuda") for I in (300, 200, 100)]
for n in range(3):
    out = torch.empty((300, 200, 100)[n], 8, dtype=torch.float64, device="cuda")
    sp.mttkrp(t, n, A, out)
t.close()
d4 = (200, 90, 40, 300)
i4, v4 = synth.tensor(95, d4, 50_000, "powerlaw")
for det in (False, True):
    t = sp.sptensor_create(d4, torch.from_numpy(i4.astype(np.int64)).cuda(),
                           torch.from_numpy(v4).cuda(), deterministic=det)
    sp.build_perm(t, -1)
    A = [torch.rand(I, 16, dtype=torch.float64, device="cuda") for I in d4]
    for n in range(4):
        out = torch.empty(d4[n], 16, dtype=torch.float64, device="cuda")
        sp.mttkrp(t, n, A, out)
    F = [torch.empty(I, 16, dtype=torch.float64, device="cuda") for I in d4]
    sp.cp_als(t, 16, 5, F, seed=1)
    t.close()
torch.cuda.synchronize()
print("sanitize case done")

# round 2 paths: forced slice / L2-window slice, options, sharded CP-ALS through a
# 1-rank communicator (peer-store and broadcast exchange), cached graph replay
t = sp.sptensor_create(dims, torch.from_numpy(idx.astype(np.int64)).cuda(),
                       torch.from_numpy(vals).cuda())
sp.build_perm(t, -1)
A = [torch.rand(I, 16, dtype=torch.float64, device="cuda") for I in dims]
for kv in ({"slice": 2}, {"slice": 2, "slice_l2_kb": 16}, {"use_copy": 0}, {"generic": 1},
           {"force_v": 1}):
    with sp.options(**kv):
        for n in range(3):
            out = torch.empty(dims[n], 16, dtype=torch.float64, device="cuda")
            sp.mttkrp(t, n, A, out)
F = [torch.empty(I, 16, dtype=torch.float64, device="cuda") for I in dims]
sp.cp_als(t, 16, 6, F, seed=1)
sp.cp_als(t, 16, 6, F, seed=1)          # replays the cached graph
os.environ["SPTK_FORCE_SHARDED"] = "1"
try:
    comm = sp.comm_create(sp.comm_unique_id(), 1, 0)
    for ex in (1, 0):
        with sp.options(exchange=ex):
            sp.cp_als(t, 16, 6, F, seed=1, comm=comm)
    comm.close()
except sp.SptkError as e:
    print("NCCL unavailable:", e)
t.close()
torch.cuda.synchronize()
print("sanitize case done (round 2 paths)")
