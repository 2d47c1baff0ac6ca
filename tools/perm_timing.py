"""Host-timed build_perm per mode (repeated) on a device-generated config."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1809_09175_b200 as sp  # noqa: E402
import synth  # noqa: E402
from synth import device  # noqa: E402

c = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "nell2"]
idx, val = device.tensor(c.seed, c.dims, c.nnz, c.dist)
t = sp.sptensor_create(c.dims, idx, val)
del idx, val
torch.cuda.empty_cache()
for rep in range(3):
    for n in range(c.N):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sp.build_perm(t, n)
        torch.cuda.synchronize()
        print(f"rep {rep} mode {n}: {1e3 * (time.perf_counter() - t0):.2f} ms", flush=True)
