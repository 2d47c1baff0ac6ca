"""Same-process A/B of option sets on the steady-state re-sort (build_perm of
one mode, CUDA events, median of REPS interleaved rounds), with the
permutations of every set checked equal to the first set's (bit-exact).
Usage: python tools/sort_ab.py config "k=v,k=v" ... ("" = defaults)"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1809_09175_b200 as sp  # noqa: E402
import synth  # noqa: E402
from synth import device  # noqa: E402
from opt_sweep import parse  # noqa: E402


def main():
    c = synth.CONFIGS[sys.argv[1]]
    sets = [parse(s) for s in sys.argv[2:]] or [{}]
    reps = int(os.environ.get("REPS", "5"))
    idx, val = device.tensor(c.seed, c.dims, c.nnz, c.dist)
    t = sp.sptensor_create(c.dims, idx, val)
    del idx, val
    torch.cuda.empty_cache()
    sp.build_perm(t, -1)
    ref = []
    for n in range(c.N):
        p = torch.empty(c.nnz, dtype=torch.int32, device="cuda")
        sp.get_perm(t, n, p)
        ref.append(p)
    times = {k: [[] for _ in range(c.N)] for k in range(len(sets))}
    for rep in range(reps):
        for k, o in enumerate(sets):
            with sp.options(**o):
                for n in range(c.N):
                    sp.build_perm(t, n)  # untimed: workspaces sized
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    torch.cuda.synchronize()
                    a.record()
                    sp.build_perm(t, n)
                    b.record()
                    torch.cuda.synchronize()
                    times[k][n].append(a.elapsed_time(b))
                    if rep == 0:
                        p = torch.empty(c.nnz, dtype=torch.int32, device="cuda")
                        sp.get_perm(t, n, p)
                        assert torch.equal(p, ref[n]), f"set {o} mode {n}: perm differs"
    for k, o in enumerate(sets):
        ms = [statistics.median(x) for x in times[k]]
        print(f"{sys.argv[1]} {o or 'defaults'}: re-sort ms/mode=" +
              " ".join(f"{m:.3f}" for m in ms) + f" sum={sum(ms):.3f}", flush=True)
    t.close()


if __name__ == "__main__":
    main()
