"""Reference CPU timing sanity check (bench.py's --impl reference arm vs its
cpu_baseline leg): per-call cost of jofc_ref::fjofc_embed at 1 / 10 / 36
iterations, inputs from oracle/workloads_ref.py (the arm) and from the
product generator (the cpu_baseline leg)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import workloads_ref  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
wl = workloads_ref.make(cfg)
R = wl.impl
t0 = time.perf_counter()
delta = wl.dense_delta()
print(f"dense_delta {time.perf_counter() - t0:.2f} s", flush=True)
x0 = wl.x0()
t0 = time.perf_counter()
R.problem(delta)
print(f"problem() {time.perf_counter() - t0:.2f} s", flush=True)
for its in (1, 10, 36, 10):
    t0 = time.perf_counter()
    r = R.fjofc_embed(delta, wl.spec, x0, 1e-300, its, parallel=True)
    sec = time.perf_counter() - t0
    print(f"{its:3d} its: {sec:.3f} s  ({sec / its:.4f} s/it; reference step_seconds sum "
          f"{r.step_seconds:.3f}, call wall {r.wall_seconds:.3f})", flush=True)
