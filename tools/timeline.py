"""Kernel timeline of CP-ALS iterations (torch.profiler / CUPTI: every kernel
and memset of the replayed graph with its device start, duration and stream)
-- the critical path the glue work reads, without nsys.
Usage: python tools/timeline.py config R iters [f64|f32] [k=v,...]
Prints the last iteration's kernels in start order: start offset, duration,
gap to the previous end on the same stream, stream, name."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_1809_09175_b200 as sp  # noqa: E402
import synth  # noqa: E402
from synth import device  # noqa: E402
from opt_sweep import parse  # noqa: E402

c = synth.CONFIGS[sys.argv[1]]
R, iters = int(sys.argv[2]), int(sys.argv[3])
dt = torch.float32 if len(sys.argv) > 4 and sys.argv[4] == "f32" else torch.float64
opts = parse(sys.argv[5]) if len(sys.argv) > 5 else {}
idx, val = device.tensor(c.seed, c.dims, c.nnz, c.dist, dtype=dt)
t = sp.sptensor_create(c.dims, idx, val)
del idx, val
torch.cuda.empty_cache()
sp.build_perm(t, -1)
F = [device.factor(c.seed_f, c.N, m, I, R, dtype=dt) for m, I in enumerate(c.dims)]
with sp.options(**opts):
    sp.cp_als(t, R, iters, F, init=F, trace=False)  # warm: caches, graph
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        sp.cp_als(t, R, iters, F, init=F, trace=False)
        torch.cuda.synchronize()
ev = []
for e in prof.events():
    if e.device_type.name != "CUDA":
        continue
    ev.append((e.time_range.start, e.time_range.end, getattr(e, "device_resource_id", 0), e.name))
ev.sort()
# one iteration: the graph replays identical iterations, so the op-name
# sequence is periodic at the end (after dropping the trailing status copy);
# take the last period
body = list(ev)
while body and ("Memcpy" in body[-1][3] or "scale_columns" in body[-1][3]):
    body.pop()  # the status copy and the final column scaling follow the last iteration
names = [x[3] for x in body]
per = next((q for q in range(2, len(names) // 2 + 1) if names[-q:] == names[-2 * q:-q]), len(names))
sel = body[-per:]
t0 = sel[0][0]
last_end = {}
busy = 0.0
print(f"{'start':>8} {'dur':>7} {'gap':>6} strm name")
for s, e_, st, n in sel:
    gap = s - last_end.get(st, s)
    last_end[st] = e_
    busy += e_ - s
    print(f"{s - t0:8.1f} {e_ - s:7.1f} {gap:6.1f} {st:4d} {n[:90]}")
span = sel[-1][1] - t0
print(f"iteration span {span:.1f} us, kernel time {busy:.1f} us ({len(sel)} ops); "
      f"{len(ev)} CUDA ops in {iters} iterations")
