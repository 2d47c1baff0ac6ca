"""Worker of tests/test_gpu_multirank.py: one rank of a torch.distributed
(NCCL) job driving libsptk's multi-GPU path -- row-range shards, shard-local
permuted copies, sharded MTTKRP with the row exchange, sharded CP-ALS -- on
a tensor every rank generates from the same seed.  Rank 0 saves the results
for the test to compare with the oracle.  Usage (torchrun):
    _multirank_worker.py <out.npz> <exchange option>"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1809_09175_b200 as sp  # noqa: E402
import synth  # noqa: E402


def main():
    out_path, exchange = sys.argv[1], int(sys.argv[2])
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    sp.set_option("exchange", exchange)
    comm = sp.comm_from_process_group()
    dims, R = (300, 257, 190), 8
    idx, vals = synth.unique_tensor(77, dims, 20000)
    t = sp.sptensor_create(dims, torch.from_numpy(idx.astype(np.int64)).cuda(),
                           torch.from_numpy(vals).cuda())
    sp.sptensor_set_shard(t, world, rank)
    sp.build_perm(t, -1)
    A = [torch.from_numpy(synth.factor(78, 3, m, I, R)).cuda() for m, I in enumerate(dims)]
    V = []
    for n in range(3):
        o = torch.full((dims[n], R), float("nan"), dtype=torch.float64, device="cuda")
        sp.mttkrp(t, n, A, o, comm=comm)
        V.append(o.cpu().numpy())
    F = [torch.empty(I, R, dtype=torch.float64, device="cuda") for I in dims]
    lam = torch.empty(R, dtype=torch.float64, device="cuda")
    res = sp.cp_als(t, R, 10, F, seed=79, comm=comm, lambda_out=lam)
    mode = sp.comm_exchange(comm)
    # every rank must hold the same replicas
    for f in F:
        g = f.clone()
        dist.broadcast(g, 0)
        assert torch.equal(f, g), "factor replicas differ between ranks"
    if rank == 0:
        np.savez(out_path, V0=V[0], V1=V[1], V2=V[2], F0=F[0].cpu().numpy(),
                 F1=F[1].cpu().numpy(), F2=F[2].cpu().numpy(), lam=lam.cpu().numpy(),
                 trace=res["trace"], mode=mode)
    t.close()
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
