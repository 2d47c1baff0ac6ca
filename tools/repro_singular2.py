"""Is LBNL's late ESINGULAR numerical?  Fresh init, one graph call of 150
iterations with the fit trace; report the first iteration that fails (via
calls of increasing length) and the fit trajectory."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1809_09175_b200 as sp  # noqa: E402
import synth  # noqa: E402
from synth import device  # noqa: E402

c = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "lbnl"]
R = int(sys.argv[3]) if len(sys.argv) > 3 else 16
idx, val = device.tensor(c.seed, c.dims, c.nnz, c.dist)
t = sp.sptensor_create(c.dims, idx, val)
del idx, val
sp.build_perm(t, -1)
for its in [int(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else "50,75,100,125,150".split(","))]:
    for mode in ("graph", "eager"):
        F = [device.factor(c.seed_f, c.N, m, I, R) for m, I in enumerate(c.dims)]
        sp.profile_enable(mode == "eager")
        lam = torch.empty(R, dtype=torch.float64, device="cuda")
        try:
            res = sp.cp_als(t, R, its, F, init=F, lambda_out=lam)
            print(f"{mode} {its}: ok fit {res['fit']:.6e}, min lambda {float(lam.min()):.3e}, "
                  f"max {float(lam.max()):.3e}", flush=True)
        except sp.SptkError as e:
            print(f"{mode} {its}: {e}", flush=True)
        sp.profile_enable(False)
