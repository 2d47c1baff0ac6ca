"""Why does bench.py's LBNL line (0.457 ms/iter) read slower than
als_sweep.py (0.4445)?  Times cp_als(K) with CUDA events under the four
combinations of {restart from the generator factors, continue} x {fit
history on, off}, interleaved.  Usage: gap_probe.py [config] [K] [rounds]"""
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1809_09175_b200 as sp  # noqa: E402
import synth  # noqa: E402
from synth import device  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "lbnl"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 50
rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 4
R = 16
c = synth.CONFIGS[name]
idx, val = device.tensor(c.seed, c.dims, c.nnz, c.dist)
t = sp.sptensor_create(c.dims, idx, val)
del idx, val
sp.build_perm(t, -1)
if os.environ.get("GP_RESORT") == "1":  # bench.py's steady-state re-sort of every mode
    for n in range(c.N):
        for _ in range(4):
            sp.build_perm(t, n)
    torch.cuda.synchronize()
F0 = [device.factor(c.seed_f, c.N, m, I, R) for m, I in enumerate(c.dims)]
F = [f.clone() for f in F0]
s = torch.cuda.current_stream()
res = {}
sp.cp_als(t, R, K, F, init=F, trace=True)
smi = None
if os.environ.get("GP_SMI") == "1":  # bench.py's clock sampler, polling every 100 ms
    smi = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,clocks.max.sm,"
                            "clocks_event_reasons.active", "--format=csv,noheader,nounits",
                            "-lms", "100"], stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
for r in range(rounds):
    for restart in (True, False):
        for trace in (True, False):
            if restart:
                for f, f0 in zip(F, F0):
                    f.copy_(f0)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            sp.cp_als(t, R, K, F, init=F, trace=trace)
            b.record(s)
            torch.cuda.synchronize()
            res.setdefault((restart, trace), []).append(a.elapsed_time(b) / K)
if smi:
    smi.terminate()
for (restart, trace), v in res.items():
    print(f"{name} K={K} resort={os.environ.get('GP_RESORT') == '1'} smi={smi is not None} restart={restart} trace={trace}: ms/iter median {statistics.median(v):.4f} "
          f"(runs {' '.join(f'{x:.4f}' for x in v)})", flush=True)
