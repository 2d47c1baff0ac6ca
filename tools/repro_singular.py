"""Repeat the bench's CP-ALS calls on a config (timed graph call, then the
profiled eager call) and count SPTK_ESINGULAR per option set.
Usage: python tools/repro_singular.py config R reps "k=v,.." ..."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import torch  # noqa: E402

import paper_1809_09175_b200 as sp  # noqa: E402
import synth  # noqa: E402
from synth import device  # noqa: E402
from opt_sweep import parse  # noqa: E402

c = synth.CONFIGS[sys.argv[1]]
R, reps = int(sys.argv[2]), int(sys.argv[3])
sets = [parse(x) for x in sys.argv[4:]] or [{}]
idx, val = device.tensor(c.seed, c.dims, c.nnz, c.dist)
t = sp.sptensor_create(c.dims, idx, val)
del idx, val
torch.cuda.empty_cache()
sp.build_perm(t, -1)
for kv in sets:
    bad = {"graph": 0, "eager": 0}
    with sp.options(**kv):
        for k in range(reps):
            F = [device.factor(c.seed_f, c.N, m, I, R) for m, I in enumerate(c.dims)]
            for mode in ("graph", "eager"):
                sp.profile_enable(mode == "eager")
                try:
                    sp.cp_als(t, R, 50, F, init=F, trace=False)
                except sp.SptkError as e:
                    bad[mode] += 1
                sp.profile_enable(False)
            torch.cuda.synchronize()
    print(f"{sys.argv[1]} {kv or 'defaults'}: {reps} reps, ESINGULAR graph {bad['graph']} eager {bad['eager']}",
          flush=True)
