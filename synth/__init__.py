"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the method (no MTTKRP, no sort, no ALS).
It only draws numbers: a counter-based generator (SURVEY.md §8(d) "The
generator spec") implemented twice from the same text -- here in numpy for
the host, and in ``synth/gen.cu`` for the device -- so that both sides see
bit-identical inputs.  ``tests/test_gpu.py::test_device_generator_matches_host`` checks the two agree.

Generator text (DESIGN.md §3 "Input recipe"):

* ``draw(seed, stream, i) = splitmix64(seed ^ (i*G) ^ (stream*H))`` with
  G = 0x9E3779B97F4A7C15, H = 0xD1B54A32D192ED03; ``u = (draw >> 11) * 2^-53``.
* streams: ``m`` (coordinate of mode m), ``N`` (value), ``N+1+m`` (factor m,
  counter ``row*R + col``).
* uniform coordinate: ``l = ((draw >> 32) * I) >> 32`` (integer, exact).
* power-law coordinate (continuous Zipf alpha=1 on [1, I+1)): ``t = u*L`` with
  ``L = log2(I+1)`` computed once on the host; ``e = floor(t)``,
  ``f = t - e``; ``y = ldexp(poly(f), e)`` where ``poly`` is a fixed degree-16
  Horner polynomial for 2^f evaluated with separate (non-fused) multiply/add;
  ``r = clamp(floor(y) - 1, 0, I-1)``; label scattering
  ``l = (a*r + b) mod I`` with ``a`` the first odd prime > I/phi coprime to I
  and ``b = floor(I/3)``.
* value ``x = 1 - u`` in (0, 1]; factor entry ``u`` in [0, 1);
  fp32 inputs are the fp64 draws rounded to nearest.
* seeds: tensor ``1809 + c``, factors ``9175 + c`` for config c (1-based).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

G_MUL = np.uint64(0x9E3779B97F4A7C15)
H_MUL = np.uint64(0xD1B54A32D192ED03)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)

# Taylor coefficients of 2^f = exp(f ln 2), degree 16 (|error| < 1e-17 on [0,1)).
# The device generator receives exactly these doubles as kernel arguments.
POW2_COEFFS = np.array([math.log(2.0) ** k / math.factorial(k) for k in range(17)],
                       dtype=np.float64)


def splitmix64(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = (x + G_MUL).astype(np.uint64)
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def draw(seed: int, stream: int, i: np.ndarray) -> np.ndarray:
    """Raw 64-bit draws for counters ``i`` (uint64 array)."""
    i = np.asarray(i, dtype=np.uint64)
    with np.errstate(over="ignore"):
        x = np.uint64(seed) ^ (i * G_MUL) ^ (np.uint64(stream) * H_MUL)
    return splitmix64(x)


def unit(d: np.ndarray) -> np.ndarray:
    """u in [0,1) from the top 53 bits (exact in fp64)."""
    return (d >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def _is_prime(n: int) -> bool:
    if n < 2:
        return False
    if n % 2 == 0:
        return n == 2
    f = 3
    while f * f <= n:
        if n % f == 0:
            return False
        f += 2
    return True


@dataclass(frozen=True)
class PowerLawParams:
    """Per-mode constants of the power-law coordinate (computed on the host only)."""
    L: float      # log2(I+1)
    a: int        # scatter multiplier (odd prime, coprime to I)
    b: int        # scatter offset

    @staticmethod
    def for_dim(I: int) -> "PowerLawParams":
        phi = (1.0 + math.sqrt(5.0)) / 2.0
        a = int(I / phi) + 1
        if a % 2 == 0:
            a += 1
        while not (_is_prime(a) and math.gcd(a, I) == 1):
            a += 2
        return PowerLawParams(L=math.log2(I + 1), a=a % I if I > 1 else 0, b=I // 3)


def coords(seed: int, mode: int, I: int, i0: int, count: int, dist: str = "uniform") -> np.ndarray:
    """Mode-``mode`` coordinates of nonzeros i0..i0+count-1 (uint32)."""
    i = np.arange(i0, i0 + count, dtype=np.uint64)
    d = draw(seed, mode, i)
    if dist == "uniform":
        with np.errstate(over="ignore"):
            l = ((d >> np.uint64(32)) * np.uint64(I)) >> np.uint64(32)
        return l.astype(np.uint32)
    if dist == "powerlaw":
        p = PowerLawParams.for_dim(I)
        u = unit(d)
        t = u * p.L
        e = np.floor(t)
        f = t - e
        y = np.full_like(f, POW2_COEFFS[-1])
        for c in POW2_COEFFS[-2::-1]:
            y = y * f
            y = y + c
        y = np.ldexp(y, e.astype(np.int32))
        r = np.floor(y).astype(np.int64) - 1
        r = np.clip(r, 0, I - 1).astype(np.uint64)
        with np.errstate(over="ignore"):
            l = (np.uint64(p.a) * r + np.uint64(p.b)) % np.uint64(I)
        return l.astype(np.uint32)
    raise ValueError(f"unknown distribution {dist!r}")


def values(seed: int, N: int, i0: int, count: int, dtype=np.float64) -> np.ndarray:
    """Values x = 1 - u in (0, 1] (stream N)."""
    i = np.arange(i0, i0 + count, dtype=np.uint64)
    x = 1.0 - unit(draw(seed, N, i))
    return x.astype(dtype)


def factor(seed_f: int, N: int, m: int, I: int, R: int, dtype=np.float64) -> np.ndarray:
    """Factor matrix A_m (I x R, row-major), entries u in [0,1) (stream N+1+m)."""
    i = np.arange(0, I * R, dtype=np.uint64)
    return unit(draw(seed_f, N + 1 + m, i)).reshape(I, R).astype(dtype)


# Integer-valued variants (the integer-exact parity pins, tests/test_gpu_exact.py):
# a draw u in [0,1) becomes the small integer 1 + floor(k*u) in {1..k}.  Both
# sides apply this same map to bit-identical draws (k*u and floor are exact
# IEEE operations), so host and device hold the same integers; every sum of
# products of them below 2^53 (fp64) / 2^24 (fp32) is exact in any order.
INT_VALUE_LEVELS = 4    # values in {1, 2, 3, 4}
INT_FACTOR_LEVELS = 3   # factor entries in {1, 2, 3}


def int_from_unit(u, k: int):
    """1 + floor(k*u) for u in [0,1) (numpy or torch arrays alike)."""
    return (u * k) // 1 + 1


def int_values(seed: int, N: int, i0: int, count: int) -> np.ndarray:
    """Integer values 1 + floor(4u), u the same draw as ``values`` (x = 1 - u)."""
    i = np.arange(i0, i0 + count, dtype=np.uint64)
    return int_from_unit(unit(draw(seed, N, i)), INT_VALUE_LEVELS)


def int_factor(seed_f: int, N: int, m: int, I: int, R: int) -> np.ndarray:
    """Integer factor 1 + floor(3u), u the same draw as ``factor``."""
    return int_from_unit(factor(seed_f, N, m, I, R), INT_FACTOR_LEVELS)


def tensor(seed: int, dims, P: int, dist: str = "uniform", i0: int = 0,
           dtype=np.float64):
    """COO tensor (idx uint32 [P, N] row-major, vals [P]) in generation order."""
    N = len(dims)
    idx = np.empty((P, N), dtype=np.uint32)
    for m, I in enumerate(dims):
        idx[:, m] = coords(seed, m, int(I), i0, P, dist)
    return idx, values(seed, N, i0, P, dtype)


def unique_tensor(seed: int, dims, P: int, dtype=np.float64):
    """Like ``tensor`` but keeps only the first occurrence of each coordinate and
    continues the counter until P distinct coordinates exist (host only; used
    where the fit is checked)."""
    N = len(dims)
    cap = int(np.prod([int(d) for d in dims], dtype=object))
    if P > cap:
        raise ValueError("P exceeds the number of cells")
    keep_idx, keep_val, seen = [], [], set()
    i0, need = 0, P
    while need > 0:
        chunk = max(2 * need, 64)
        idx, vals = tensor(seed, dims, chunk, "uniform", i0, np.float64)
        lin = np.zeros(chunk, dtype=object)
        for m in range(N):
            lin = lin * int(dims[m]) + idx[:, m].astype(object)
        for k in range(chunk):
            key = lin[k]
            if key in seen:
                continue
            seen.add(key)
            keep_idx.append(idx[k])
            keep_val.append(vals[k])
            need -= 1
            if need == 0:
                break
        i0 += chunk
    idx = np.array(keep_idx, dtype=np.uint32).reshape(P, N)
    return idx, np.array(keep_val, dtype=np.float64).astype(dtype)


def planted_tensor(seed: int, dims, R: int, support):
    """Sparse tensor that is EXACTLY a rank-R Kruskal tensor [[mu; B_0..B_{N-1}]].

    Column r of B_m is supported on ``support[m]`` rows; mode-0 supports of
    different columns are disjoint, so every coordinate belongs to exactly one
    component and coordinates are unique.  Returns (idx uint32 [P,N], vals f64
    [P], mu [R], B list of dense I_m x R arrays).  Host only.
    """
    N = len(dims)
    rng_i = 0

    def u(stream, n):
        nonlocal rng_i
        out = unit(draw(seed, 100 + stream, np.arange(rng_i, rng_i + n, dtype=np.uint64)))
        rng_i += n
        return out

    if support[0] * R > dims[0]:
        raise ValueError("mode-0 supports must be disjoint: need support[0]*R <= dims[0]")
    B = [np.zeros((int(I), R)) for I in dims]
    rows = []
    for m in range(N):
        rows_m = []
        for r in range(R):
            if m == 0:
                sel = np.arange(r * support[0], (r + 1) * support[0])
            else:
                # support rows: distinct, chosen by a seeded shuffle
                keys = u(m, int(dims[m]))
                sel = np.sort(np.argsort(keys, kind="stable")[: support[m]])
            B[m][sel, r] = 0.5 + u(10 + m, len(sel))
            rows_m.append(sel)
        rows.append(rows_m)
    mu = 1.0 + u(50, R)
    idx_list, val_list = [], []
    for r in range(R):
        grids = np.meshgrid(*[rows[m][r] for m in range(N)], indexing="ij")
        coords_r = np.stack([g.reshape(-1) for g in grids], axis=1)
        v = np.full(coords_r.shape[0], mu[r])
        for m in range(N):
            v = v * B[m][coords_r[:, m], r]
        idx_list.append(coords_r)
        val_list.append(v)
    idx = np.concatenate(idx_list).astype(np.uint32)
    vals = np.concatenate(val_list)
    # storage order: a seeded shuffle so no mode is presorted
    order = np.argsort(u(99, idx.shape[0]), kind="stable")
    return idx[order], vals[order], mu, B


@dataclass(frozen=True)
class Config:
    """One BASELINE.json config as a concrete synthetic workload."""
    number: int
    name: str
    dims: tuple
    nnz: int
    ranks: tuple
    dtypes: tuple
    dist: str = "uniform"
    unique: bool = False
    extra: dict = field(default_factory=dict)

    @property
    def seed(self) -> int:
        return 1809 + self.number

    @property
    def seed_f(self) -> int:
        return 9175 + self.number

    @property
    def N(self) -> int:
        return len(self.dims)


CONFIGS = {
    "tiny": Config(1, "tiny", (100, 80, 60), 2000, (8,), ("f64",), unique=True),
    "lbnl": Config(2, "lbnl", (1600, 4200, 1600, 4200, 868000), 1_700_000, (16,), ("f64",)),
    "nell2": Config(3, "nell2", (12000, 9200, 28800), 77_000_000, (16, 64), ("f64", "f32")),
    "delicious": Config(4, "delicious", (532000, 17_000_000, 2_500_000, 1400), 140_000_000,
                        (16,), ("f64",), dist="powerlaw"),
    "amazon": Config(5, "amazon", (4_800_000, 1_800_000, 1_800_000), 1_700_000_000,
                     (16,), ("f64",)),
    # the paper's own synthetic CP-ALS / bandwidth-vs-R workload:
    # "30K x 40K x 50K with 10M nonzeros placed randomly", R = 128 and R in [8, 256]
    "paper_synth": Config(6, "paper_synth", (30000, 40000, 50000), 10_000_000, (128,), ("f64",)),
    # VAST-like shape (not a BASELINE config): a length-2 mode, the
    # short-mode / contention study of SURVEY §8(f) NEXT-4
    "vast_shape": Config(7, "vast_shape", (165000, 11000, 2, 100, 89), 26_000_000, (16,), ("f64",)),
}
