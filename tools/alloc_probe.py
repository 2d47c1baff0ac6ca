"""Host time of large cudaMalloc calls in this process (PYTORCH_NO_CUDA_MEMORY_CACHING=1:
every torch.empty is a cudaMalloc, every del a cudaFree).  Usage:
  PYTORCH_NO_CUDA_MEMORY_CACHING=1 python tools/alloc_probe.py [prewarm_GB]
prewarm_GB > 0: allocate and free that much first (does it make the later
allocations cheaper?)"""
import os
import sys
import time

import torch

pre = float(sys.argv[1]) if len(sys.argv) > 1 else 0.0
torch.cuda.init()
torch.empty(1, device="cuda")
torch.cuda.synchronize()
if pre > 0:
    t0 = time.perf_counter()
    x = torch.empty(int(pre * (1 << 30)), dtype=torch.uint8, device="cuda")
    x.zero_()
    torch.cuda.synchronize()
    del x
    torch.cuda.synchronize()
    print(f"prewarm {pre} GB: {1e3 * (time.perf_counter() - t0):.2f} ms")
bufs = []
for k in range(6):
    t0 = time.perf_counter()
    bufs.append(torch.empty(int(1.23 * (1 << 30)), dtype=torch.uint8, device="cuda"))
    torch.cuda.synchronize()
    print(f"alloc {k} 1.23 GB: {1e3 * (time.perf_counter() - t0):.3f} ms", flush=True)
