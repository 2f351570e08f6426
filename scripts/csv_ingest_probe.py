"""CSV ingest rate: jofc_load_problem_files on headerless CSVs (m = 2,
n = 5000, %.17g text) vs the reference's load_dissimilarities.  Diagnostic."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1502_03391_b200 as jg  # noqa: E402
from paper_1502_03391_b200 import workloads  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 5000
wl = workloads.make(5, n=n)
dense = wl.dense_delta()
root = "/dev/shm" if os.path.isdir("/dev/shm") else "/tmp"
paths = []
for l in range(wl.m):
    p = os.path.join(root, f"jofc_csv_probe_{l}.csv")
    np.savetxt(p, dense[l], delimiter=",", fmt="%.17g")
    paths.append(p)
size = sum(os.path.getsize(p) for p in paths)
dev = jg.Device(0)
jg.load_dissimilarities(paths, device=dev)
t0 = time.perf_counter()
for _ in range(3):
    jg.load_dissimilarities(paths, device=dev)
sec = (time.perf_counter() - t0) / 3
print(f"ours: {sec * 1e3:.1f} ms per load, {size / sec / 1e9:.2f} GB/s of CSV text "
      f"({size / 1e6:.0f} MB)")
try:
    from oracle.oracle import Reference
    R = Reference()
    t0 = time.perf_counter()
    R.load_dissimilarities(paths)
    sec = time.perf_counter() - t0
    print(f"reference: {sec * 1e3:.1f} ms per load, {size / sec / 1e9:.2f} GB/s")
except Exception as e:  # noqa: BLE001
    print("reference unavailable:", e)
for p in paths:
    os.remove(p)
