"""Same-process A/B of launch options on CP-ALS ms/iteration (graph replay,
median of REPS interleaved rounds of `iters` iterations after a warm-up).
Usage: python tools/als_sweep.py config R f64|f32 "k=v,k=v" ... ("" = defaults)"""
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
    name, R, dts = sys.argv[1], int(sys.argv[2]), sys.argv[3]
    sets = [parse(s) for s in sys.argv[4:]] or [{}]
    reps, iters = int(os.environ.get("REPS", "3")), int(os.environ.get("ITERS", "20"))
    dt = torch.float64 if dts == "f64" else torch.float32
    c = synth.CONFIGS[name]
    idx, val = device.tensor(c.seed, c.dims, c.nnz, c.dist, dtype=dt)
    t = sp.sptensor_create(c.dims, idx, val)
    del idx, val
    torch.cuda.empty_cache()
    sp.build_perm(t, -1)
    F = [device.factor(c.seed_f, c.N, m, I, R, dtype=dt) for m, I in enumerate(c.dims)]
    res = [[] for _ in sets]
    for _ in range(reps):
        for si, kv in enumerate(sets):
            with sp.options(**kv):
                sp.cp_als(t, R, 4, F, init=F, trace=False)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                a.record()
                sp.cp_als(t, R, iters, F, init=F, trace=False)
                b.record()
                torch.cuda.synchronize()
                res[si].append(a.elapsed_time(b) / iters)
    for si, kv in enumerate(sets):
        print(f"{name} R={R} {dts} {kv or 'defaults'}: CP-ALS ms/iter median {statistics.median(res[si]):.4f} "
              f"(runs {' '.join(f'{x:.4f}' for x in res[si])})", flush=True)
    t.close()


if __name__ == "__main__":
    main()
