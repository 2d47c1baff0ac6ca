"""Intermittent SPTK_ESINGULAR on LBNL: numerical or a race?  Build once,
then run cp_als(K iterations) from the generator factors `reps` times and
report failures and the spread of the final fit (a deterministic trajectory
differs only by atomic-order rounding).  Options come from SPTK_* env vars.
Usage: race_hunt.py [config] [K] [reps] [R]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1809_09175_b200 as sp  # noqa: E402
import synth  # noqa: E402
from synth import device  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "lbnl"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 10
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 30
R = int(sys.argv[4]) if len(sys.argv) > 4 else 16
c = synth.CONFIGS[name]
idx, val = device.tensor(c.seed, c.dims, c.nnz, c.dist)
t = sp.sptensor_create(c.dims, idx, val, deterministic=os.environ.get("RH_DET") == "1")
del idx, val
sp.build_perm(t, -1)
F0 = [device.factor(c.seed_f, c.N, m, I, R) for m, I in enumerate(c.dims)]
F = [f.clone() for f in F0]
fails, fits, lams, traces, hashes = 0, [], [], [], set()
import hashlib  # noqa: E402
lam = torch.empty(R, dtype=torch.float64, device="cuda")
for r in range(reps):
    for f, f0 in zip(F, F0):
        f.copy_(f0)
    torch.cuda.synchronize()
    try:
        res = sp.cp_als(t, R, K, F, init=F, lambda_out=lam, trace=True)
        fits.append(res["fit"])
        traces.append(list(res["trace"]))
        hashes.add(hashlib.sha1(b"".join(f.cpu().numpy().tobytes() for f in F)).hexdigest())
        lams.append(float(lam.min()))
    except sp.SptkError as e:
        fails += 1
        print(f"  rep {r}: {e}", flush=True)
env = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith(("SPTK_", "RH_"))) or "defaults"
if fits:
    print(f"{name} K={K} [{env}]: {fails}/{reps} failed; fit min {min(fits):.9e} max {max(fits):.9e}; "
          f"min-lambda range [{min(lams):.3e}, {max(lams):.3e}]; {len(hashes)} distinct factor bit patterns",
          flush=True)
else:
    print(f"{name} K={K} [{env}]: {fails}/{reps} failed", flush=True)
if traces:  # where do the odd trajectories leave the common one?
    ref = max(set(tuple(x) for x in traces), key=lambda x: sum(tuple(y) == x for y in traces))
    for k, tr in enumerate(traces):
        d = [i for i, (a, b) in enumerate(zip(tr, ref)) if abs(a - b) > 1e-9 * abs(b)]
        if d:
            print(f"  odd trajectory: leaves the common one at iteration {d[0]}: "
                  f"{tr[d[0]]:.9e} vs {ref[d[0]]:.9e}", flush=True)
