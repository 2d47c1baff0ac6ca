"""The paper's bandwidth-vs-R experiment (Fig. mttkrp_bandwidth) and
synthetic CP-ALS timing (Fig. cpals_time) on B200, on the paper's
own synthetic tensor (30K x 40K x 50K, 10M random nonzeros, fp64).
Prints, per R in [8, 256] step 8: MTTKRP ms summed over modes, the paper's
bandwidth model ((dR+3) s_r + d s_o) P / t with s_o = 8, its ratio to
the measured HBM copy peak, and B_model GB/s; then CP-ALS R=128, 10 iterations.
Usage: python tools/rsweep.py [Rmax] [step]"""
import json
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
    rmax = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    step = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    try:
        peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:
        peak = 6650.0
    c = synth.CONFIGS["paper_synth"]
    idx, val = device.tensor(c.seed, c.dims, c.nnz, c.dist)
    t = sp.sptensor_create(c.dims, idx, val)
    del idx, val
    sp.build_perm(t, -1)
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    for R in range(step, rmax + 1, step):
        A = [device.factor(c.seed_f, c.N, m, I, R) for m, I in enumerate(c.dims)]
        outs = [torch.empty((I, R), dtype=torch.float64, device="cuda") for I in c.dims]
        for n in range(c.N):
            sp.mttkrp(t, n, A, outs[n])
        a, b = ev(), ev()
        reps = 10
        a.record()
        for _ in range(reps):
            for n in range(c.N):
                sp.mttkrp(t, n, A, outs[n])
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / reps
        paper = sum(metrics.paper_bandwidth(c.N, R, c.nnz, 8, 8, ms * 1e-3 / c.N) for _ in c.dims) / c.N
        bm = sum(metrics.b_model(c.N, c.nnz, R, I, 8) for I in c.dims) / (ms * 1e-3) / 1e9
        print(json.dumps({"R": R, "mttkrp_ms_all_modes": round(ms, 4),
                          "paper_model_GBps": round(paper / 1e9, 1),
                          "paper_model_pct_of_copy_peak": round(100 * paper / 1e9 / peak, 1),
                          "b_model_GBps": round(bm, 1)}), flush=True)
    R = 128
    F = [torch.empty((I, R), dtype=torch.float64, device="cuda") for I in c.dims]
    sp.cp_als(t, R, 2, F, seed=c.seed_f)
    sp.profile_reset()
    sp.profile_enable(True)
    a, b = ev(), ev()
    a.record()
    res = sp.cp_als(t, R, 10, F, seed=c.seed_f)
    b.record()
    torch.cuda.synchronize()
    sp.profile_enable(False)
    prof = sp.profile_read()
    tot = a.elapsed_time(b)
    print(json.dumps({"cp_als_R": R, "iters": res["iters"], "total_ms": round(tot, 3),
                      "ms_per_iter": round(tot / 10, 3),
                      "mttkrp_share": round(prof["mttkrp_ms"] / tot, 3),
                      "fit": res["fit"]}), flush=True)


if __name__ == "__main__":
    main()
