"""Time the FIRST build_perm(-1) after ingest (what bench.py reports as
setup.build_perm_all_ms), K times in one process (tensor destroyed and the
caching allocator emptied in between).  Usage: python tools/first_build.py [config] [K]
SPTK_DEBUG_SETUP=1 prints the phase breakdown (synchronising between phases)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1809_09175_b200 as sp  # noqa: E402
import synth  # noqa: E402
from synth import device  # noqa: E402

c = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "nell2"]
K = int(sys.argv[2]) if len(sys.argv) > 2 else 3
for k in range(K):
    idx, val = device.tensor(c.seed, c.dims, c.nnz, c.dist)
    t = sp.sptensor_create(c.dims, idx, val)
    del idx, val
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    h0 = time.perf_counter()
    a.record()
    sp.build_perm(t, -1)
    b.record()
    torch.cuda.synchronize()
    print(f"{c.name} first build_perm(-1) #{k}: device {a.elapsed_time(b):.2f} ms, host "
          f"{1e3 * (time.perf_counter() - h0):.2f} ms, tensor {sp.sptensor_device_bytes(t) / 1e9:.2f} GB",
          flush=True)
    t.close()
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
