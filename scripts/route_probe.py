"""Whole-solve device time of one config through the graph route vs the single-launch
persistent route (JOFC_PERSISTENT=0/1), no per-pass events.  python scripts/route_probe.py CFG"""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1502_03391_b200 as jg  # noqa: E402
from paper_1502_03391_b200 import workloads  # noqa: E402
from paper_1502_03391_b200._capi import check  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
wl = workloads.make(cfg)
dev = jg.Device(0)
dev.upload_features(wl.in_features)
x0 = torch.from_numpy(wl.x0()).cuda()
ptr = C.cast(x0.data_ptr(), C.POINTER(C.c_double))
lib = dev.lib
stream = torch.cuda.ExternalStream(dev.stream)


def solve():
    check(lib.jofc_fjofc_enqueue(dev.h, C.byref(wl.spec.c()), wl.d, ptr, 1e-300, wl.iterations))


for _ in range(3):
    solve()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 10
e0.record(stream)
for _ in range(reps):
    solve()
e1.record(stream)
e1.synchronize()
ms = e0.elapsed_time(e1) / reps
print(f"cfg{cfg} persistent={os.environ.get('JOFC_PERSISTENT', 'auto')} "
      f"fidelity={os.environ.get('JOFC_FIDELITY', 'auto')}: {ms:.3f} ms per solve, "
      f"{wl.iterations / ms * 1e3:.1f} it/s")
