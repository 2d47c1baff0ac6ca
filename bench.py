#!/usr/bin/env python
"""Benchmark: sparse MTTKRP HBM GB/s & CP-ALS ms/iter at R=16 (BASELINE.json).

One "step" = one CP-ALS iteration over the resident tensor: an MTTKRP for
every mode plus the ALS glue (Gram/Hadamard/Cholesky/solve/normalise/fit) and,
for N > 1 ranks, the NCCL exchange of each updated factor -- every row of
SURVEY.md §8(a) that repeats per iteration (a3-a9).  Ingest (a1) and
build_perm (a2) are one-time setup, timed separately and reported in
"setup".  Default workload: the NELL-2-shaped config (BASELINE configs[2],
where the metric's HBM-fraction target is stated), R=16, fp64.

value = B_model bytes of the step's MTTKRPs (per-gather north
star byte model) / device time per step, whole job; ms_per_step = CP-ALS
ms/iteration.  Launch: `python bench.py --gpus N --steps K --warmup W`
(N > 1 under torch.distributed.run, one rank per GPU, NCCL).
`--impl reference` times the CPU oracle (the reference arm for this tier).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from paper_1809_09175_b200 import metrics  # noqa: E402

METRIC = "sparse MTTKRP HBM GB/s & CP-ALS ms/iter at R=16, 1/2/4/8 B200"
FALLBACK_HBM = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback (GB/s)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="sptk", choices=["sptk", "reference"])
    ap.add_argument("--config", default="nell2", choices=list(synth.CONFIGS))
    ap.add_argument("--rank", type=int, default=16)
    ap.add_argument("--dtype", default="f64", choices=["f64", "f32"])
    ap.add_argument("--cpu-seconds", type=float, default=12.0,
                    help="target CPU seconds for the oracle baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--layout", default="sorted", choices=["sorted", "perm_gather"],
                    help="sorted: records materialised in perm order at build_perm (default); "
                         "perm_gather: the paper's literal gather through perm_n")
    return ap.parse_args()


def peaks():
    try:
        j = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return FALLBACK_HBM, "fallback (B200_PROFILING.md)"


def _profile_json(name: str):
    try:
        return json.load(open(os.path.join(ROOT, "profiles", name)))
    except Exception:
        return {}


def limiter_for(workload_key: str):
    """What ncu showed bounds the MTTKRP launch (committed capture), if any."""
    return _profile_json("ncu_limiter.json").get(workload_key)


def traffic_for(workload_key: str):
    """ncu DRAM bytes per MTTKRP launch from the committed capture, if any
    (keyed <config>_R<R>_<dtype>[_perm_gather]: the layout changes the bytes)."""
    return _profile_json("ncu_traffic.json").get(workload_key)


def gather_ceilings(row_bytes: int):
    """Measured random-row gather ceilings (tools/ceilings.cu ->
    profiles/ceilings.json) for rows of `row_bytes`: L1-resident table (the
    L1 data-pipe rate: no gather can beat it), L2-resident (L2 -> SM) and
    HBM-resident tables."""
    j = _profile_json("ceilings.json")
    rb = min((64, 128, 256, 512), key=lambda b: abs(b - row_bytes))

    def v(k):
        e = j.get(k)
        return e["value"] if isinstance(e, dict) else None
    # the slice MTTKRP's own access mix (16 B record + one L1-resident and one
    # L2-resident 128 B row per nonzero, no arithmetic, perfect window hits):
    # the best grid of tools/ceilings.cu's pair_gather runs
    pair = [v(k) for k in j if k.startswith(f"pair_gather_l1_l2_{rb}_")] if j else []
    pair = [x for x in pair if x]
    return {"row_bytes": rb, "l1_resident": v(f"gather_l1_l1_{rb}"),
            "l2_resident": v(f"gather_l2_nol1_{rb}"), "l2_resident_l1alloc": v(f"gather_l2_l1_{rb}"),
            "hbm_resident": v(f"gather_hbm_nol1_{rb}"), "hbm_read": v("hbm_read"),
            "slice_mix": (max(pair) if pair else None),
            "source": "profiles/ceilings.json (tools/ceilings.cu)" if j else None}


# ------------------------------------------------------------------ clocks
REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
           0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
           0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
           0x100: "display_clock_setting"}


class ClockSampler:
    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.proc = None
        self.thread = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 3:
                try:
                    self.samples.append((float(parts[0]), float(parts[1]), int(parts[2], 16),
                                         time.perf_counter()))
                except ValueError:
                    pass

    def wait_first(self, timeout=5.0):
        t0 = time.perf_counter()
        while self.proc and not self.samples and time.perf_counter() - t0 < timeout:
            time.sleep(0.02)

    def mark(self, which):
        setattr(self, which, time.perf_counter())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)

    def summary(self):
        t0, t1 = getattr(self, "t_start", None), getattr(self, "t_end", None)
        sel = [s for s in self.samples if t0 is not None and t0 <= s[3] <= t1 + 0.15]
        window = "timed region"
        if not sel and self.samples and t0 is not None:   # region shorter than the 100 ms period
            sel = sorted(self.samples, key=lambda s: abs(s[3] - 0.5 * (t0 + t1)))[:2]
            window = "nearest samples to the timed region"
        if not sel:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        mask = 0
        for s in sel:
            mask |= s[2]
        reasons = [name for bit, name in REASONS.items() if mask & bit and name != "gpu_idle"]
        return {"sm_mhz": statistics.median(s[0] for s in sel),
                "sm_max_mhz": max(s[1] for s in sel), "reasons": reasons,
                "samples": len(sel), "window": window}


# ------------------------------------------------------------------ oracle leg
class OracleSample:
    """The oracle (row-owned OpenMP form, as it stands) on a bounded sample of
    the workload: the first P_s nonzeros of the same generator stream with
    full-size factors.  The oracle's own counting-sort perms are built once
    (not timed, like build_perm on the GPU side)."""

    def __init__(self, c, R: int, np_dtype, Ps: int):
        import oracle
        self.oracle, self.c, self.R, self.Ps = oracle, c, R, Ps
        self.s_v = np.dtype(np_dtype).itemsize
        self.A = [synth.factor(c.seed_f, c.N, m, int(I), R).astype(np_dtype).astype(np.float64)
                  for m, I in enumerate(c.dims)]
        self.idx, vals = synth.tensor(c.seed, c.dims, Ps, c.dist)
        self.vals = vals.astype(np_dtype).astype(np.float64)
        self.perms = [oracle.perm(self.idx, n, int(I)) for n, I in enumerate(c.dims)]
        self.bytes = sum(metrics.b_model(c.N, Ps, R, int(I), self.s_v) for I in c.dims)

    def step(self):
        """MTTKRP of every mode; returns (seconds, threads used)."""
        t0 = time.perf_counter()
        nt = 1
        for n in range(self.c.N):
            _, nt = self.oracle.mttkrp_omp(self.c.dims, self.idx, self.vals, self.A, n,
                                           self.perms[n][0], self.perms[n][1])
        return time.perf_counter() - t0, nt

    def describe(self, dt):
        c = self.c
        return (f"first {self.Ps:,} of {c.nnz:,} nonzeros of the {c.name} generator stream, "
                f"full-size factors, MTTKRP of all {c.N} modes per step (oracle_mttkrp_omp: "
                f"counting-sort perm + row-owned OpenMP; perm not timed); {dt:.2f} s per step")


def sized_sample(c, R, np_dtype, target_s: float) -> OracleSample:
    """Calibrate P_s so that one oracle step takes about target_s seconds."""
    probe = OracleSample(c, R, np_dtype, min(c.nnz, 500_000))
    dt, _ = probe.step()
    if dt >= target_s or probe.Ps >= c.nnz:
        return probe
    Ps = int(min(c.nnz, probe.Ps * target_s / max(dt, 1e-4)))
    return OracleSample(c, R, np_dtype, Ps)


def oracle_sample_rate(c, R: int, target_s: float, np_dtype):
    smp = sized_sample(c, R, np_dtype, target_s)
    dt, nt = smp.step()
    return smp.bytes / dt / 1e9, nt, smp.describe(dt), smp.Ps, dt


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    c = synth.CONFIGS[args.config]
    np_dtype = np.float64 if args.dtype == "f64" else np.float32
    per_step = max(0.5, min(10.0, 90.0 / max(1, args.steps + args.warmup)))
    smp = sized_sample(c, args.rank, np_dtype, per_step)
    times, cores = [], 1
    for k in range(args.warmup + args.steps):
        dt, cores = smp.step()
        if k >= args.warmup:
            times.append(dt)
    dt = statistics.median(times)
    v = smp.bytes / dt / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "GB/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3,
        "higher_is_better": True, "dtype": args.dtype, "data": "synthetic",
        "config": {"workload": workload_name(c, args.rank, args.dtype)},
        "cpu_baseline": {"value": v, "unit": "GB/s", "cores": cores, "kind": "oracle",
                         "sample": smp.describe(dt)},
        "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def l2_note(c, R, dtype, s_v):
    rec = c.nnz * (32 if (s_v == 8 and c.N > 2) or c.N > 3 else 16)
    fac = sum(I * R * s_v for I in c.dims)
    where = ("L2-resident (gathers served from the 126 MB L2)" if fac < 100e6
             else "larger than L2 (gathers served from HBM)")
    return (f"inputs larger than L2, no flush needed: records {rec / 1e9:.2f} GB + perms "
            f"{c.N * c.nnz * 4 / 1e9:.2f} GB stream per step vs 126 MB L2; factor matrices "
            f"{fac / 1e6:.1f} MB, {where}")


def workload_name(c, R, dtype):
    d = "x".join(str(x) for x in c.dims)
    return f"{c.name}-shaped {c.N}-way {d}, {c.nnz:,} nnz, {c.dist}, R={R}, {dtype}"


# ------------------------------------------------------------------ GPU leg
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    import paper_1809_09175_b200 as sp
    from synth import device as sdev

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    # SPTK_FORCE_SHARDED=1 under torchrun with one rank exercises the N>1 path
    # (process group, NCCL bootstrap, sharded ALS) on a single GPU
    distributed = world > 1 or bool(os.environ.get("SPTK_FORCE_SHARDED")) and "RANK" in os.environ
    if distributed:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    comm = sp.comm_from_process_group() if distributed else None

    c = synth.CONFIGS[args.config]
    R = args.rank
    tdt = torch.float64 if args.dtype == "f64" else torch.float32
    s_v = 8 if args.dtype == "f64" else 4
    stream = torch.cuda.current_stream()

    # ---- setup: generate (device), ingest, build perms (timed, not in the step)
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    # warm the setup path once on a small tensor of the same order and dtype:
    # the first use of each kernel in a process loads its module (CUDA lazy
    # loading), which made the first build_perm vary 18-38 ms run to run
    # (profiles/r02/first_build.log); the timed setup below is then the
    # tensor's own cost (the cold one is reported as well)
    h0 = time.perf_counter()
    wdims = tuple(min(int(I), 4096) for I in c.dims)
    wi, wv = sdev.tensor(c.seed + 1000, wdims, 1 << 16, c.dist, dtype=tdt)
    wt = sp.sptensor_create(wdims, wi, wv, perm_gather=args.layout == "perm_gather")
    sp.build_perm(wt, -1)
    wF = [sdev.factor(c.seed_f, c.N, m, I, R, dtype=tdt) for m, I in enumerate(wdims)]
    sp.cp_als(wt, R, 4, wF, init=wF, trace=False)
    torch.cuda.synchronize()
    wt.close()
    del wi, wv, wF
    warm_ms = 1e3 * (time.perf_counter() - h0)
    e0, e1, e2 = ev(), ev(), ev()
    e0.record()
    idx_d, val_d = sdev.tensor(c.seed, c.dims, c.nnz, c.dist, dtype=tdt)
    e1.record()
    t = sp.sptensor_create(c.dims, idx_d, val_d, perm_gather=args.layout == "perm_gather")
    if world > 1:  # each rank keeps permuted copies of its own row ranges only
        sp.sptensor_set_shard(t, world, rank)
    e2.record()
    torch.cuda.synchronize()
    del idx_d, val_d
    torch.cuda.empty_cache()  # return the COO staging to the driver (perm copies need it)
    # the paper's preprocessing (Table `sorting_cost`): one
    # build_perm of every mode right after ingest -- sorts from the keys the
    # ingest pass emitted, allocations and the permuted copies included
    a, b = ev(), ev()
    h0 = time.perf_counter()
    a.record()
    sp.build_perm(t, -1)
    b.record()
    torch.cuda.synchronize()
    perm_all_ms, perm_all_host_ms = a.elapsed_time(b), 1e3 * (time.perf_counter() - h0)
    perm_ms = []   # steady-state re-sort per mode (keys extracted from the records)
    free_b, total_b = torch.cuda.mem_get_info()
    # skipped when the sort workspace no longer fits beside the copies (the
    # re-sort would evict them: Amazon shape on one GPU)
    for n in (range(c.N) if free_b > 16 * c.nnz + (8 << 30) else []):
        sp.build_perm(t, n)  # untimed: the first call per mode sizes the workspaces
        torch.cuda.synchronize()
        reps = []  # median of three: one re-sort is ~1.5 ms, a host hiccup is not
        for _ in range(3):
            a, b = ev(), ev()
            a.record()
            sp.build_perm(t, n)
            b.record()
            torch.cuda.synchronize()
            reps.append(a.elapsed_time(b))
        perm_ms.append(sorted(reps)[1])
    F = [sdev.factor(c.seed_f, c.N, m, I, R, dtype=tdt) for m, I in enumerate(c.dims)]
    # every measured pass starts from these generator factors, so each one
    # times the same iterations 1..K
    F0 = [f.clone() for f in F]

    def reset_factors():
        for f, f0 in zip(F, F0):
            f.copy_(f0)
    dev_bytes = sp.sptensor_device_bytes(t)

    # per-rank share of the work (row-range sharding) for the byte model
    bounds, pos, rowptrs = [], [], []
    for n, I in enumerate(c.dims):
        rp = torch.empty(I + 1, dtype=torch.int32, device="cuda")
        sp.get_rowptr(t, n, rp)
        rph = rp.cpu().numpy().view(np.uint32)
        rowptrs.append(rph)
        bd = sp.partition_rows(rph, world)
        bounds.append(bd)
        pos.append((int(rph[bd[rank]]), int(rph[bd[rank + 1]])))
    bm_total = sum(metrics.b_model(c.N, c.nnz, R, I, s_v) for I in c.dims)
    # B_comp: compulsory HBM bytes -- the nonzeros' indices and
    # values, the perm, each distinct factor row touched once, the output
    nonempty = [int(np.count_nonzero(np.diff(rp_n.astype(np.int64)))) for rp_n in rowptrs]
    bc_modes = [metrics.b_comp(c.N, c.nnz, R, c.dims[n],
                               sum(nonempty[m] for m in range(c.N) if m != n), s_v)
                for n in range(c.N)]
    bm_rank = sum(metrics.b_model(c.N, pos[n][1] - pos[n][0], R,
                                  int(bounds[n][rank + 1] - bounds[n][rank]), s_v)
                  for n in range(c.N))

    def barrier():
        if world > 1:
            dist.barrier()

    with ClockSampler(local) as clk:
        clk.wait_first()
        # warm-up: W CP-ALS iterations (>= 3)
        sp.cp_als(t, R, max(3, args.warmup), F, init=F, comm=comm, trace=False)
        reset_factors()
        torch.cuda.synchronize()

        # ---- timed region: K consecutive CP-ALS iterations (one call continues the
        # factors in place; the library replays the iteration as a CUDA graph),
        # device time with CUDA events on the launching stream
        sp.profile_enable(False)
        sp.profile_reset()
        barrier()
        torch.cuda.synchronize()
        clk.mark("t_start")
        start, end = ev(), ev()
        start.record(stream)
        res = sp.cp_als(t, R, args.steps, F, init=F, comm=comm, trace=True)
        end.record(stream)
        torch.cuda.synchronize()
        clk.mark("t_end")
        barrier()
        launches = sp.profile_read()["kernel_launches"]
        # ---- roofline pass: the same K iterations with the library's per-launch
        # CUDA events around every MTTKRP kernel (eager launches: events inside a
        # graph cannot be timed)
        sp.profile_reset()
        sp.profile_enable(True)
        reset_factors()
        torch.cuda.synchronize()
        pa, pb = ev(), ev()
        pa.record(stream)
        sp.cp_als(t, R, args.steps, F, init=F, comm=comm, trace=False)
        pb.record(stream)
        torch.cuda.synchronize()
        sp.profile_enable(False)
        prof = sp.profile_read()
        time.sleep(0.15)
    ms = start.elapsed_time(end) / args.steps
    ms_t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    value = bm_total / (ms_max * 1e-3) / 1e9
    ms_eager = pa.elapsed_time(pb) / args.steps

    # dominant kernel (MTTKRP) roofline on this rank.  achieved = ALGORITHMIC
    # bytes per launch (B_comp: compulsory HBM bytes) / mean launch
    # time; the per-gather north-star model B_model is reported beside it as
    # frac_model (it counts L2/L1-served factor rows as memory traffic)
    mttkrp_ms_launch = prof["mttkrp_ms"] / max(1, prof["mttkrp_launches"])
    t_launch = mttkrp_ms_launch * 1e-3
    bc_launch = sum(bc_modes) / c.N / world   # rank share (row-range shards)
    bm_launch = bm_rank / c.N
    achieved = bc_launch / t_launch / 1e9
    peak, peak_src = peaks()
    key = f"{args.config}_R{R}_{args.dtype}" + ("_perm_gather" if args.layout == "perm_gather" else "")
    traffic = traffic_for(key)
    ncu = limiter_for(key)
    gathered = c.nnz * (c.N - 1) * R * s_v / world   # per launch, counted per gather
    ceil = gather_ceilings(R * s_v)
    gather_rate = gathered / t_launch / 1e9
    binding = None
    if ncu and ncu.get("l1tex_data_pipe_lsu_wavefronts_pct") is not None:
        binding = {"unit": "L1 data pipe (LSU wavefronts: every gathered factor row, hit or miss)",
                   "frac": ncu["l1tex_data_pipe_lsu_wavefronts_pct"] / 100.0,
                   "lts_frac": (ncu.get("lts_throughput_pct") or 0) / 100.0 or None,
                   "source": ncu.get("source")}
    elif ncu:
        binding = {"unit": ncu.get("limiter"), "frac": None, "source": ncu.get("source")}

    # ---- end to end through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        Fh = [torch.empty((I, R), dtype=tdt).pin_memory() for I in c.dims]
        for m in range(c.N):
            Fh[m].copy_(F0[m].cpu())
        for _ in range(2):
            sp.cp_als(t, R, 1, Fh, init=Fh, comm=comm, trace=False)
        barrier()
        torch.cuda.synchronize()
        a, b = ev(), ev()
        a.record(stream)
        for _ in range(args.steps):
            sp.cp_als(t, R, 1, Fh, init=Fh, comm=comm, trace=False)
        b.record(stream)
        torch.cuda.synchronize()
        e_ms = a.elapsed_time(b) / args.steps
        et = torch.tensor([e_ms], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(et, op=dist.ReduceOp.MAX)
        fbytes = sum(I * R * s_v for I in c.dims)
        e2e = {"value": bm_total / (float(et.item()) * 1e-3) / 1e9, "unit": "GB/s",
               "ms_per_step": float(et.item()), "h2d_bytes_per_step": fbytes,
               "d2h_bytes_per_step": fbytes + 8,
               "path": "sptk_cp_als(max_iters=1) with pinned HOST factor buffers: H2D of all "
                       "factors, one ALS iteration, D2H of the factors and the fit, per step; "
                       "the tensor is ingested once (setup)"}

    # ---- CPU baseline: the oracle on a bounded sample (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        gbs, cores, desc, Ps, dt = oracle_sample_rate(
            c, R, args.cpu_seconds, np.float64 if args.dtype == "f64" else np.float32)
        cpu = {"value": gbs, "unit": "GB/s", "cores": cores, "kind": "oracle", "sample": desc}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms_max,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": args.dtype, "data": "synthetic",
            "config": {
                "workload": workload_name(c, R, args.dtype), "dims": list(c.dims),
                "nnz": c.nnz, "R": R, "dist": c.dist, "seed": c.seed, "seed_f": c.seed_f,
                "step": "one CP-ALS iteration (MTTKRP all modes + glue + exchange); the K timed "
                        "iterations run in one sptk_cp_als(max_iters=K) call continuing the factors",
                "layout": args.layout,
                "parallelism": f"row-range shard x{world}" if world > 1 else "single GPU",
                "l2": l2_note(c, R, args.dtype, s_v),
            },
            "cp_als_ms_per_iter": ms_max,
            "cp_als_ms_per_iter_eager": ms_eager,
            "fit_after_timed_iters": res["fit"],
            "mttkrp_ms_per_mode": mttkrp_ms_launch,
            "b_model_bytes_per_step": bm_total,
            "gflops": sum(metrics.flops(c.N, c.nnz, R) for _ in c.dims) / (ms_max * 1e-3) / 1e9,
            "setup": {"generate_ms": e0.elapsed_time(e1), "create_ms": e1.elapsed_time(e2),
                      "process_warmup_ms": warm_ms,
                      "build_perm_all_ms": perm_all_ms, "build_perm_all_host_ms": perm_all_host_ms,
                      "resort_ms_per_mode": perm_ms,
                      # the paper's Table `sorting_cost` ratio: the permutation sorts
                      # (steady state, no allocation) per CP-ALS iteration
                      "sort_to_iteration_ratio": (sum(perm_ms) / ms_max) if perm_ms else None,
                      # everything build_perm does the first time (allocations, the
                      # permuted copies and their secondary sorts) per iteration
                      "setup_to_iteration_ratio": perm_all_host_ms / ms_max,
                      "tensor_device_bytes": dev_bytes},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": ncu.get("kernel") if ncu else
                                   "MTTKRP launch (permuted copy; slice, warp-cooperative or per-group kernel chosen per mode)",
                         "bytes_algorithmic": "B_comp per launch = P(N*4+s_v) + 4P + sum_{m!=n} U_m*R*s_v "
                                              "+ I_n*R*s_v (SURVEY 8(d), U_m = nonempty rows), mean over modes",
                         "bytes_algorithmic_per_launch": bc_launch,
                         "peak_source": peak_src,
                         # the same launch measured by the DRAM bytes ncu saw it move
                         "frac_dram": (traffic / t_launch / 1e9 / peak) if traffic else None,
                         # the north star's per-gather byte model: > 1 when the
                         # gathered rows are served from L2/L1
                         "frac_model": bm_launch / t_launch / 1e9 / peak,
                         "bytes_model_per_launch": bm_launch,
                         # what actually bounds the launch (ncu) and the gather rate
                         # against the measured random-row gather ceilings
                         "binding": binding,
                         "gather": {"achieved": gather_rate, "unit": "GB/s",
                                    "bytes_per_launch": gathered,
                                    "ceilings": ceil,
                                    "frac_of_l1_resident": (gather_rate / ceil["l1_resident"]
                                                            if ceil.get("l1_resident") else None),
                                    "frac_of_slice_mix": (gather_rate / ceil["slice_mix"]
                                                          if ceil.get("slice_mix") else None)},
                         "timing": "per-launch CUDA events in a second K-iteration pass "
                                   "(eager launches), mean over all MTTKRP launches"},
            "clocks": clk.summary(),
            "gpu_launches": launches,
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    t.close()
    if comm is not None:
        comm.close()
    if distributed:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
