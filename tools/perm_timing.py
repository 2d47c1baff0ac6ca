"""Host-timed build_perm per mode (repeated; argv[2] repetitions, default 3) on a device-generated config.
The tensor is created twice: the first pass includes one-time costs (lazy
module loading, first allocations); the second shows build_perm right after
ingest (sort keys emitted by the pack kernel) and then repeated calls (keys
released, extracted from the records per mode)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1809_09175_b200 as sp  # noqa: E402
import synth  # noqa: E402
from synth import device  # noqa: E402

c = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "nell2"]
for tensor_pass in range(2):
    idx, val = device.tensor(c.seed, c.dims, c.nnz, c.dist)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    t = sp.sptensor_create(c.dims, idx, val)
    torch.cuda.synchronize()
    print(f"pass {tensor_pass} create: {1e3 * (time.perf_counter() - t0):.2f} ms "
          f"(device bytes {sp.sptensor_device_bytes(t) / 1e9:.2f} GB)", flush=True)
    del idx, val
    torch.cuda.empty_cache()
    for rep in range(int(sys.argv[2]) if len(sys.argv) > 2 else 3):
        for n in range(c.N):
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0 = time.perf_counter()
            a.record()
            sp.build_perm(t, n)
            t1 = time.perf_counter()
            b.record()
            torch.cuda.synchronize()
            print(f"pass {tensor_pass} rep {rep} mode {n}: {1e3 * (time.perf_counter() - t0):.2f} ms "
                  f"(device {a.elapsed_time(b):.2f} ms, host call {1e3 * (t1 - t0):.2f} ms)", flush=True)
    t0 = time.perf_counter()
    t.close()
    torch.cuda.synchronize()
    print(f"pass {tensor_pass} destroy: {1e3 * (time.perf_counter() - t0):.2f} ms", flush=True)
