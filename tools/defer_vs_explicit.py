"""Deferred vs explicit column normalisation on one bit-reproducible tensor
(deterministic MTTKRP): after K = 1..Kmax iterations from the generator
factors, how far apart are lambda and the normalised factors, and how well
conditioned is every mode's Gamma (host fp64 eigenvalues of the Hadamard
product of the other modes' Gram matrices)?  Usage: defer_vs_explicit.py [config] [Kmax] [R]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1809_09175_b200 as sp  # noqa: E402
import synth  # noqa: E402
from synth import device  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "lbnl"
Kmax = int(sys.argv[2]) if len(sys.argv) > 2 else 8
R = int(sys.argv[3]) if len(sys.argv) > 3 else 16
c = synth.CONFIGS[name]
idx, val = device.tensor(c.seed, c.dims, c.nnz, c.dist)
t = sp.sptensor_create(c.dims, idx, val, deterministic=True)
del idx, val
sp.build_perm(t, -1)
F0 = [device.factor(c.seed_f, c.N, m, I, R) for m, I in enumerate(c.dims)]
F = [f.clone() for f in F0]
lam = torch.empty(R, dtype=torch.float64, device="cuda")


def run(K, deferred):
    sp.set_option("deferred_norm", deferred)
    for f, f0 in zip(F, F0):
        f.copy_(f0)
    torch.cuda.synchronize()
    try:
        res = sp.cp_als(t, R, K, F, init=F, lambda_out=lam, trace=True)
    except sp.SptkError as e:
        return None, str(e), None, None
    return list(res["trace"]), lam.cpu().numpy().copy(), [f.cpu().numpy().copy() for f in F], res


for K in range(1, Kmax + 1):
    te, le, fe, _ = run(K, 0)
    td, ld, fd, _ = run(K, 1)
    if te is None or td is None:
        print(f"K={K}: explicit {le if te is None else 'ok'}; deferred {ld if td is None else 'ok'}")
        continue
    dl = np.max(np.abs(ld - le)) / np.max(np.abs(le))
    df = max(float(np.max(np.abs(a - b))) for a, b in zip(fd, fe))
    grams = [a.T @ a for a in fe]
    conds = []
    for n in range(c.N):
        g = np.ones((R, R))
        for m in range(c.N):
            if m != n:
                g = g * grams[m]
        ev = np.linalg.eigvalsh(g)
        conds.append(ev[-1] / max(ev[0], 1e-300))
    print(f"K={K}: fit e {te[-1]:.12e} d {td[-1]:.12e}; |dlambda|/max {dl:.2e}; max|dA| {df:.2e}; "
          f"lambda e min {le.min():.3e} max {le.max():.3e}; d min {ld.min():.3e} max {ld.max():.3e}; "
          f"cond(Gamma_n) {' '.join(f'{x:.1e}' for x in conds)}", flush=True)
    if K == Kmax or dl > 1e-6:
        print("   lambda e:", " ".join(f"{x:.4e}" for x in le))
        print("   lambda d:", " ".join(f"{x:.4e}" for x in ld))
sp.set_option("deferred_norm", 1)
