"""sptensor_create from HOST buffers (pageable numpy and pinned torch) on a
BASELINE config; prints the ingest time and the device footprint.
Usage: python tools/ingest_timing.py [config]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1809_09175_b200 as sp  # noqa: E402
import synth  # noqa: E402
from synth import device  # noqa: E402

c = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "nell2"]
idx_d, val_d = device.tensor(c.seed, c.dims, c.nnz, c.dist)
idx_h = idx_d.cpu().numpy().astype(np.int64)          # pageable host, int64 like a file reader
val_h = val_d.cpu().numpy()
idx_p = torch.from_numpy(idx_h).pin_memory()
val_p = torch.from_numpy(val_h).pin_memory()
del idx_d, val_d
torch.cuda.empty_cache()
for name, (i, v) in {"pageable numpy": (idx_h, val_h), "pinned torch": (idx_p, val_p)}.items():
    for rep in range(2):
        torch.cuda.synchronize()
        free0 = torch.cuda.mem_get_info()[0]
        t0 = time.perf_counter()
        t = sp.sptensor_create(c.dims, i, v)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        gb = (i.nbytes if hasattr(i, "nbytes") else i.numel() * 8) + v.nbytes if hasattr(v, "nbytes") else 0
        print(f"{name} rep {rep}: {1e3 * dt:.1f} ms, {(idx_h.nbytes + val_h.nbytes) / dt / 1e9:.1f} GB/s of input, "
              f"device bytes {sp.sptensor_device_bytes(t) / 1e9:.2f} GB", flush=True)
        t.close()
