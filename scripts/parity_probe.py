"""Worst stress-trace and final-X differences of full-size solves against the reference
(oracle/_ref), printed rather than asserted: for judging an experimental build
(JOFC_GPU_LIB=...) against the 1e-10 / 1e-8 tolerances.

python scripts/parity_probe.py [cfg ...]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1502_03391_b200 as jg  # noqa: E402
from oracle.oracle import Reference, Spec  # noqa: E402  (the checker)
from paper_1502_03391_b200 import workloads  # noqa: E402

R = Reference()
dev = jg.Device(0)
for cfg in [int(a) for a in sys.argv[1:]] or [2, 5, 4, 3]:
    wl = workloads.make(cfg)
    delta, x0 = wl.dense_delta(), wl.x0()
    spec_o = Spec.general_(wl.spec.general) if wl.general_weights else Spec.uniform(wl.w)
    ref = R.fjofc_embed(delta, spec_o, x0, 1e-300, wl.iterations, parallel=True)
    opt = jg.SolveOptions(dim=wl.d, eps=1e-300, max_iterations=wl.iterations,
                          init=jg.InitKind.provided, init_config=x0)
    r = jg.fjofc_embed(jg.OmnibusProblem(list(delta), validate=False), wl.spec, opt, device=dev)
    k = min(len(r.stress_trace), len(ref.trace))
    worst = max(abs(a - b) / abs(b) for a, b in zip(r.stress_trace[:k], ref.trace[:k]))
    ex = float(np.linalg.norm(r.config - ref.x) / np.linalg.norm(ref.x))
    print(f"cfg{cfg} [{os.path.basename(os.environ.get('JOFC_GPU_LIB', 'default'))}]: iterations "
          f"{r.iterations}/{ref.iterations}, worst trace rel err {worst:.3e}, X rel err {ex:.3e}",
          flush=True)
