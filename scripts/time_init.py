"""Time the GPU averaged_procrustes_init at a config size."""
import sys
import time
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1502_03391_b200 as jg  # noqa: E402
from paper_1502_03391_b200 import workloads  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
wl = workloads.make(cfg)
dev = jg.Device(0)
dev.upload_features(wl.in_features)
import ctypes as C, numpy as np  # noqa: E401,E402
from paper_1502_03391_b200._capi import check, dptr  # noqa: E402
out = np.empty((wl.m, wl.n, wl.d))
t0 = time.perf_counter()
check(dev.lib.jofc_init_averaged_procrustes(dev.h, wl.d, dptr(out)))
print(f"cfg{cfg} averaged_procrustes_init n={wl.n} m={wl.m} d={wl.d}: "
      f"{time.perf_counter() - t0:.2f} s, launches {dev.launches()}")
