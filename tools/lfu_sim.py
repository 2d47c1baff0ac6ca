"""Ideal LFU row-cache simulation for the Delicious-shaped MTTKRP (profiles/r02/lfu_delicious.txt).
Usage: PYTHONPATH=. python tools/lfu_sim.py"""
import numpy as np, synth, time
c = synth.CONFIGS["delicious"]
P = c.nnz
counts = []
t0=time.time()
for m, I in enumerate(c.dims):
    cnt = np.zeros(I, dtype=np.int64)
    for i0 in range(0, P, 20_000_000):
        n = min(20_000_000, P - i0)
        cnt += np.bincount(synth.coords(c.seed, m, I, i0, n, c.dist), minlength=I)
    counts.append(cnt)
    print(m, I, "nonempty", int((cnt>0).sum()), "max", int(cnt.max()), time.time()-t0, flush=True)

for n in range(4):
    others = [m for m in range(4) if m != n]
    allc = np.concatenate([counts[m] for m in others])
    allc = np.sort(allc[allc > 0])[::-1]
    tot = allc.sum()
    distinct = len(allc)
    for mb in (32, 64, 100, 126):
        k = mb * 2**20 // 128
        hit = allc[:k].sum() - min(k, distinct)  # compulsory first touch
        miss = tot - hit
        print(f"mode {n}: gathers {tot/1e6:.0f}M distinct rows {distinct/1e6:.2f}M  ideal static {mb}MB: misses {miss/1e6:.1f}M lines = {miss*128/1e9:.2f} GB")
