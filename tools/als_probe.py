"""CP-ALS on a config for a few iterations (for ncu launch lists).
Usage: python tools/als_probe.py config R iters [f64|f32]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1809_09175_b200 as sp  # noqa: E402
import synth  # noqa: E402
from synth import device  # noqa: E402

c = synth.CONFIGS[sys.argv[1]]
R, iters = int(sys.argv[2]), int(sys.argv[3])
dt = torch.float32 if len(sys.argv) > 4 and sys.argv[4] == "f32" else torch.float64
idx, val = device.tensor(c.seed, c.dims, c.nnz, c.dist, dtype=dt)
t = sp.sptensor_create(c.dims, idx, val)
del idx, val
torch.cuda.empty_cache()  # return the COO input to the driver (room for the copies)
sp.build_perm(t, -1)
F = [torch.empty((I, R), dtype=dt, device="cuda") for I in c.dims]
res = sp.cp_als(t, R, iters, F, seed=c.seed_f)
torch.cuda.synchronize()
print(res)
