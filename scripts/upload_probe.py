"""Host -> device upload of a dense C3 problem: raw pinned H2D bandwidth vs
jofc_set_problem (2-D chunk copies + pack kernels).  Diagnostic only."""
import ctypes as C
import time

import numpy as np
import torch

import paper_1502_03391_b200 as jg
from paper_1502_03391_b200 import workloads
from paper_1502_03391_b200._capi import _dp, check, dptr

wl = workloads.make(3)
delta = wl.dense_delta()
cudart = torch.cuda.cudart()
assert int(cudart.cudaHostRegister(delta.ctypes.data, delta.nbytes, 0)) == 0
src = torch.from_numpy(delta.reshape(-1)[: 400_000_000])  # 3.2 GB registered
dst = torch.empty(src.numel(), dtype=torch.float64, device="cuda")
for _ in range(2):
    dst.copy_(src, non_blocking=True)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(3):
    dst.copy_(src, non_blocking=True)
torch.cuda.synchronize()
sec = (time.perf_counter() - t0) / 3
print(f"raw H2D (registered host, 1-D): {src.numel() * 8 / sec / 1e9:.1f} GB/s")
del dst
dev = jg.Device(0)
ptrs = (_dp * wl.m)(*[dptr(delta[l]) for l in range(wl.m)])
check(dev.lib.jofc_set_problem(dev.h, wl.m, wl.n, ptrs, 0))
ts = []
for _ in range(3):
    t0 = time.perf_counter()
    check(dev.lib.jofc_set_problem(dev.h, wl.m, wl.n, ptrs, 0))
    ts.append(time.perf_counter() - t0)
sec = min(ts)
print(f"jofc_set_problem: {sec * 1e3:.1f} ms (min of 3: {[round(t * 1e3, 1) for t in ts]}), "
      f"{3283397120 / sec / 1e9:.1f} GB/s of the uploaded bytes")
