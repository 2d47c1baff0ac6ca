"""Build the in-tree shared objects for sm_100a (no GPU needed: nvcc cross-compiles).

* ``paper_1809_09175_b200/libsptk.so`` -- the product (csrc/*.cu), C ABI in include/sptk.h
* ``synth/libsynth.so``              -- the device input generator (test/bench input only)

Objects are rebuilt when their source or any header is newer.  Usage:
``python -m paper_1809_09175_b200.build [--force]``.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(PKG, "build")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
         "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include")]
LIB = os.path.join(PKG, "libsptk.so")


def _nccl_device_include():
    """Include dir of the NCCL runtime torch ships (2.28+: nccl_device.h, the
    symmetric-memory window and device-communicator API used by comm.cu), or
    None -- comm.cu then builds without the fused exchange (NCCL broadcast)."""
    try:
        import importlib.util
        spec = importlib.util.find_spec("nvidia.nccl")
        for d in (spec.submodule_search_locations or []):
            inc = os.path.join(d, "include")
            if os.path.exists(os.path.join(inc, "nccl_device.h")):
                return inc
    except Exception:
        pass
    return None


def _extra_flags(src):
    if os.path.basename(src) == "comm.cu":
        inc = _nccl_device_include()
        if inc:
            return ["-I", inc, "-DSPTK_NCCL_DEVICE_API=1"]
    return []


SYNTH_SRC = os.path.join(ROOT, "synth", "gen.cu")
SYNTH_LIB = os.path.join(ROOT, "synth", "libsynth.so")


def _newest(paths):
    return max((os.path.getmtime(p) for p in paths), default=0.0)


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("build failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)
    return r.stdout + r.stderr


def build(force: bool = False, verbose: bool = False, jobs: int | None = None) -> str:
    os.makedirs(OBJ, exist_ok=True)
    sources = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    headers = glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "sptk.h")]
    hdr_time = _newest(headers)
    todo, objs = [], []
    for src in sources:
        obj = os.path.join(OBJ, os.path.basename(src)[:-3] + ".o")
        objs.append(obj)
        if force or not os.path.exists(obj) or os.path.getmtime(obj) < max(
                os.path.getmtime(src), hdr_time):
            todo.append((src, obj))
    ptxas = ["-Xptxas", "-v"] if verbose else []
    with cf.ThreadPoolExecutor(max_workers=jobs or os.cpu_count() or 4) as ex:
        futs = {ex.submit(_run, [NVCC, *ARCH, *FLAGS, *_extra_flags(src), *ptxas, "-c", src, "-o",
                                 obj + ".tmp"]): (src, obj)
                for src, obj in todo}
        for f in cf.as_completed(futs):
            src, obj = futs[f]
            out = f.result()
            os.replace(obj + ".tmp", obj)
            if verbose and out:
                print(f"== {os.path.basename(src)}\n{out}")
    if force or todo or not os.path.exists(LIB) or os.path.getmtime(LIB) < _newest(objs):
        _run([NVCC, *ARCH, "-shared", "-o", LIB + ".tmp", *objs, "-ldl"])
        os.replace(LIB + ".tmp", LIB)
    if force or not os.path.exists(SYNTH_LIB) or os.path.getmtime(SYNTH_LIB) < os.path.getmtime(SYNTH_SRC):
        _run([NVCC, *ARCH, *FLAGS, "-shared", "-o", SYNTH_LIB + ".tmp", SYNTH_SRC])
        os.replace(SYNTH_LIB + ".tmp", SYNTH_LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
