"""Device time of jofc_oos_batch (fixed 100 updates, inputs resident on the GPU) for a
range of batch shapes: the persistent solve (JOFC_OOS_KERNEL unset) vs the per-update
kernels (JOFC_OOS_KERNEL=3)."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1502_03391_b200 as jg  # noqa: E402
from paper_1502_03391_b200._capi import check  # noqa: E402

dev = jg.Device(0)
lib = dev.lib
P = C.POINTER(C.c_double)
rng = np.random.default_rng(5)
shapes = [tuple(int(v) for v in s.split(",")) for s in sys.argv[1:]] or [
    (1, 2, 5000, 3), (8, 2, 5000, 3), (148, 2, 5000, 3), (300, 2, 5000, 3), (450, 2, 5000, 3),
    (600, 2, 5000, 3), (800, 2, 5000, 3), (1000, 2, 5000, 3), (2000, 2, 5000, 3),
    (1, 2, 200000, 3), (300, 2, 20000, 5), (1000, 2, 20000, 5)]
stream = torch.cuda.ExternalStream(dev.stream)
for k, m, n, d in shapes:
    x = torch.from_numpy(rng.normal(size=(m, n, d))).cuda()
    od = torch.from_numpy(np.abs(rng.normal(size=(k, m, n))) + 1.0).cuda()
    y0 = torch.from_numpy(rng.normal(size=(k, m, d))).cuda()
    yo = torch.empty_like(y0)

    def run():
        check(lib.jofc_oos_batch(dev.h, k, m, n, d, C.cast(x.data_ptr(), P), C.cast(od.data_ptr(), P),
                                 0.5, C.cast(y0.data_ptr(), P), 1e-300, 100, 1,
                                 C.cast(yo.data_ptr(), P), None, None))
    run()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    e0.record(stream)
    for _ in range(reps):
        run()
    e1.record(stream)
    e1.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"{os.environ.get('JOFC_OOS_KERNEL', '4')} k={k} m={m} n={n} d={d}: {ms:.3f} ms "
          f"per 100-update solve")
