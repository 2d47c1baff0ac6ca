"""Same-process A/B of launch options on a BASELINE config (device-generated
inputs, one tensor): each option set is timed per mode (mean of 20 launches
after 3 warm-ups, CUDA events), the sets interleaved over `REPS` rounds so
clock drift hits them alike; prints the median per set.
Usage: python tools/opt_sweep.py config R f64|f32 "k=v,k=v" "k=v" ...
("" = defaults).  Options: include/sptk.h sptk_set_option."""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1809_09175_b200 as sp  # noqa: E402
import synth  # noqa: E402
from synth import device  # noqa: E402


def parse(spec):
    kv = {}
    for part in filter(None, spec.split(",")):
        k, v = part.split("=")
        kv[k.strip()] = int(v)
    return kv


def main():
    name, R, dts = sys.argv[1], int(sys.argv[2]), sys.argv[3]
    sets = [parse(s) for s in sys.argv[4:]] or [{}]
    reps = int(os.environ.get("REPS", "3"))
    dt = torch.float64 if dts == "f64" else torch.float32
    c = synth.CONFIGS[name]
    idx, val = device.tensor(c.seed, c.dims, c.nnz, c.dist, dtype=dt)
    t = sp.sptensor_create(c.dims, idx, val)
    del idx, val
    torch.cuda.empty_cache()
    sp.build_perm(t, -1)
    A = [device.factor(c.seed_f, c.N, m, I, R, dtype=dt) for m, I in enumerate(c.dims)]
    outs = [torch.empty((I, R), dtype=dt, device="cuda") for I in c.dims]
    res = [[[] for _ in range(c.N)] for _ in sets]
    disp = [[""] * c.N for _ in sets]
    for _ in range(reps):
        for si, kv in enumerate(sets):
            with sp.options(**kv):
                for n in range(c.N):
                    for _ in range(3):
                        sp.mttkrp(t, n, A, outs[n])
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record()
                    for _ in range(20):
                        sp.mttkrp(t, n, A, outs[n])
                    b.record()
                    torch.cuda.synchronize()
                    res[si][n].append(a.elapsed_time(b) / 20)
                    disp[si][n] = sp.last_dispatch()
    for si, kv in enumerate(sets):
        ms = [statistics.median(x) for x in res[si]]
        print(f"{name} R={R} {dts} {kv or 'defaults'}: ms/mode={' '.join(f'{x:.3f}' for x in ms)} "
              f"sum={sum(ms):.3f}  [{'; '.join(disp[si])}]", flush=True)
    t.close()


if __name__ == "__main__":
    main()
