"""Wall time of a typical user solve (eps = 1e-6, max_iterations = 1000) that
converges early: the synchronous API stops enqueuing once the device says done."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1502_03391_b200 as jg  # noqa: E402
from paper_1502_03391_b200 import workloads  # noqa: E402

for cfg, n in ((1, None), (5, 2000)):
    wl = workloads.make(cfg, n=n)
    prob = jg.OmnibusProblem(list(wl.dense_delta()), validate=False)
    dev = jg.Device(0)
    opt = jg.SolveOptions(dim=wl.d, eps=1e-6, max_iterations=1000, init=jg.InitKind.provided,
                          init_config=wl.x0())
    jg.fjofc_embed(prob, wl.spec, opt, device=dev)  # warm-up
    t0 = time.perf_counter()
    r = jg.fjofc_embed(prob, wl.spec, opt, device=dev)
    dt = time.perf_counter() - t0
    print(f"cfg{cfg} n={wl.n}: {r.iterations} iterations ({r.terminated.name}), "
          f"{dt * 1e3:.2f} ms, launches {dev.launches()}")

# one out-of-sample point with the default options (eps 1e-6, 1000 iterations)
import numpy as np  # noqa: E402

wl = workloads.make(5, n=2000)
x = np.random.default_rng(0).normal(size=(wl.m, wl.n, wl.d))
od = np.abs(np.random.default_rng(1).normal(size=(wl.m, wl.n))) + 1.0
dev = jg.Device(0)
jg.oos_embed(x, od, 0.5, jg.OosOptions(), 7, device=dev)
t0 = time.perf_counter()
res = jg.oos_embed(x, od, 0.5, jg.OosOptions(), 7, device=dev)
print(f"oos_embed n={wl.n}: {res.iterations} iterations ({res.terminated.name}), "
      f"{(time.perf_counter() - t0) * 1e3:.2f} ms, launches {dev.launches()}")
