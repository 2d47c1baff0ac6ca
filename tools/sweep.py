"""MTTKRP sweep on a BASELINE config (device-generated inputs): layouts
(LAYOUTS=sorted,perm_gather,atomic -- atomic is the paper's VerA/VerB
storage-order traversal), worker shapes (VARIANTS) and block lengths (RUNS).
Usage: python tools/sweep.py [config] [R] [f64|f32]
Prints ms per mode (mean of 20 launches after warm-up, CUDA events)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1809_09175_b200 as sp  # noqa: E402
import synth  # noqa: E402
from paper_1809_09175_b200 import metrics  # noqa: E402
from synth import device  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "nell2"
    R = int(sys.argv[2]) if len(sys.argv) > 2 else 16
    dt = torch.float64 if (len(sys.argv) < 4 or sys.argv[3] == "f64") else torch.float32
    variants = [int(v) for v in os.environ.get("VARIANTS", "0,1").split(",")]
    runs = [int(r) for r in os.environ.get("RUNS", "128,256,512,1024").split(",")]
    layouts = os.environ.get("LAYOUTS", "sorted").split(",")
    c = synth.CONFIGS[name]
    idx, val = device.tensor(c.seed, c.dims, c.nnz, c.dist, dtype=dt)
    A = [device.factor(c.seed_f, c.N, m, I, R, dtype=dt) for m, I in enumerate(c.dims)]
    outs = [torch.empty((I, R), dtype=dt, device="cuda") for I in c.dims]
    s_v = 8 if dt == torch.float64 else 4
    tensors = {}
    for layout in layouts:
        tensors[layout] = sp.sptensor_create(c.dims, idx, val, perm_gather=layout == "perm_gather")
    del idx, val                 # the COO input is not needed after ingest (frees HBM for
    torch.cuda.empty_cache()     # the permuted copies, as in bench.py)
    for layout in layouts:
        t = tensors.pop(layout)
        if layout != "atomic":
            sp.build_perm(t, -1)
        call = sp.mttkrp_atomic if layout == "atomic" else sp.mttkrp
        for v in (variants if layout == "sorted" else [-1]):
            for run in (runs if layout != "atomic" else [0]):
                sp.set_tuning(v, run)
                ms = []
                for n in range(c.N):
                    for _ in range(3):
                        call(t, n, A, outs[n])
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record()
                    for _ in range(20):
                        call(t, n, A, outs[n])
                    b.record()
                    torch.cuda.synchronize()
                    ms.append(a.elapsed_time(b) / 20)
                bm = sum(metrics.b_model(c.N, c.nnz, R, I, s_v) for I in c.dims)
                print(f"{name} R={R} {str(dt)[6:]} {layout:11s} variant={v} run={run:5d}  "
                      f"ms/mode={' '.join(f'{x:.3f}' for x in ms)}  sum={sum(ms):.3f}  "
                      f"B_model GB/s={bm / sum(ms) / 1e6:.0f}", flush=True)
        t.close()
        sp.set_tuning(-2, -2)


if __name__ == "__main__":
    main()
