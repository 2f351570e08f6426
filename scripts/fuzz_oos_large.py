"""One-off randomised sweep of the out-of-sample batch solve at large in-sample counts (the
multi-chunk ring of the persistent launch, many point groups), both routes, against the
oracle on a sample of the batch's points.  The suite's sweep stops at n = 2049.

python scripts/fuzz_oos_large.py [seed [cases]]
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1502_03391_b200 as jg  # noqa: E402
from oracle.oracle import Port  # noqa: E402  (the checker)


def rel_fro(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(b))


def main():
    seed = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    cases = int(sys.argv[2]) if len(sys.argv) > 2 else 16
    dev = jg.Device(0)
    worst_y = worst_s = 0.0
    for case in range(cases):
        rng = np.random.default_rng(seed * 104729 + case)
        m = int(rng.integers(1, 5))
        n = int(rng.choice([2050, 3000, 5000, 8191, 12000, 20000]))
        d = int(rng.integers(1, 11))
        k = int(rng.choice([1, 33, 500, 1500]))
        its = int(rng.integers(2, 12))
        x = rng.normal(size=(m, n, d))
        yt = rng.normal(size=(k, m, d))
        od = np.empty((k, m, n))
        for l in range(m):
            g = (x[l] * x[l]).sum(1)[None, :] + (yt[:, l] * yt[:, l]).sum(1)[:, None]
            od[:, l, :] = np.sqrt(np.maximum(g - 2.0 * yt[:, l] @ x[l].T, 0.0))
        od = np.abs(od + 0.05 * rng.normal(size=od.shape))
        y0 = rng.normal(size=(k, m, d))
        w = float(rng.uniform(0.1, 1.5))
        sample = np.unique(np.linspace(0, k - 1, min(k, 24)).astype(int))
        yr, trr, itr = Port().oos_batch(x, od[sample], w, y0[sample], 1e-300, its, fixed=True)
        for route in (1, 2):
            t0 = time.perf_counter()
            dev.set_oos_route(route)
            try:
                y, tr, it = jg.oos_embed_batch(x, od, w, y0, jg.OosOptions(1e-300, its),
                                               fixed_iterations=True, device=dev)
            finally:
                dev.set_oos_route(0)
            ey = max(rel_fro(y[q], yr[j]) for j, q in enumerate(sample))
            es = max(float(np.max(np.abs(tr[q] - trr[j]) / np.abs(trr[j])))
                     for j, q in enumerate(sample))
            ok = ey < 1e-8 and es < 1e-10 and all(it[q] == itr[j] for j, q in enumerate(sample))
            worst_y, worst_s = max(worst_y, ey), max(worst_s, es)
            print(f"case {case} route {route}: m={m} n={n} d={d} k={k} its={its} y {ey:.2e} "
                  f"trace {es:.2e} {'ok' if ok else 'MISMATCH'} ({time.perf_counter() - t0:.1f} s)",
                  flush=True)
            if not ok:
                sys.exit(1)
    print(f"all {cases} cases ok (both routes): worst y rel err {worst_y:.2e}, worst trace rel err "
          f"{worst_s:.2e}")
    dev.close()


if __name__ == "__main__":
    main()
