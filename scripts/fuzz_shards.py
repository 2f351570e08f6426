"""One-off randomised sweep of the sharded data path on ONE GPU: W contexts own the block
ranges jofc_set_shard gives them, partial products go through the all-reduce hook
(ThreadGroup: host-side reduction), every rank must reproduce the unsharded solve.  The suite
(tests/test_gpu_shards.py) runs worlds 2 and 3 at n = 700; this sweeps worlds 2..8, n up to
5000 (both solve routes), every d, the three weight families.

python scripts/fuzz_shards.py [seed [cases]]
"""
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1502_03391_b200 as jg  # noqa: E402
from paper_1502_03391_b200.dist import ThreadGroup  # noqa: E402


def main():
    seed = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    cases = int(sys.argv[2]) if len(sys.argv) > 2 else 24
    dev0 = jg.Device(0)
    worst = 0.0
    for case in range(cases):
        rng = np.random.default_rng(seed * 7919 + case)
        world = int(rng.choice([2, 3, 4, 5, 7, 8]))
        m = int(rng.integers(1, 5))
        n = int(rng.choice([129, 300, 517, 1100, 2300, 3100, 5000]))
        d = int(rng.integers(1, 11))
        its = int(rng.integers(2, 9))
        z = rng.normal(size=(n, 3))
        delta = []
        for _ in range(m):
            f = z + 0.2 * rng.normal(size=(n, 3))
            g = (f * f).sum(1)
            dm = np.sqrt(np.maximum(g[:, None] + g[None, :] - 2.0 * f @ f.T, 0.0))
            dm = 0.5 * (dm + dm.T)
            np.fill_diagonal(dm, 0.0)
            delta.append(dm)
        kind = int(rng.integers(0, 3))
        if kind == 0:
            spec = jg.WeightSpec.uniform(float(rng.uniform(0.1, 2.0)))
        elif kind == 1:
            spec = jg.WeightSpec.product(rng.uniform(0.5, 2.0, size=m), float(rng.uniform(0.5, 1.5)))
        else:
            a = rng.uniform(0.2, 1.0, size=(m, m))
            spec = jg.WeightSpec.general(0.5 * (a + a.T))
        x0 = rng.normal(size=(m, n, d))
        prob = jg.OmnibusProblem(delta, validate=False)
        opt = jg.SolveOptions(dim=d, eps=1e-300, max_iterations=its, init=jg.InitKind.provided,
                              init_config=x0)
        t0 = time.perf_counter()
        single = jg.fjofc_embed(prob, spec, opt, device=dev0)
        group = ThreadGroup(world)
        results, errors = [None] * world, []

        def run(rank):
            try:
                dev = jg.Device(0, shard=(rank, world))
                dev.set_allreduce(group.hook_for(rank, "cuda:0"))
                results[rank] = jg.fjofc_embed(prob, spec, opt, device=dev)
                dev.close()
            except Exception as e:  # noqa: BLE001
                errors.append(e)
                group.bar.abort()

        threads = [threading.Thread(target=run, args=(r,)) for r in range(world)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        if errors:
            print(f"case {case}: world={world} m={m} n={n} d={d}: {errors[0]!r}")
            sys.exit(1)
        ex = es = 0.0
        for res in results:
            ok_it = res.iterations == single.iterations
            ex = max(ex, float(np.linalg.norm(res.config - single.config)
                               / np.linalg.norm(single.config)))
            es = max(es, max(abs(a - b) / abs(b)
                             for a, b in zip(res.stress_trace, single.stress_trace)))
            if not ok_it:
                ex = float("inf")
        worst = max(worst, ex, es)
        ok = ex < 1e-11 and es < 1e-11
        print(f"case {case}: world={world} m={m} n={n} d={d} its={its} kind={kind} X {ex:.2e} "
              f"trace {es:.2e} {'ok' if ok else 'MISMATCH'} ({time.perf_counter() - t0:.1f} s)",
              flush=True)
        if not ok:
            sys.exit(1)
    print(f"all {cases} cases ok: worst rel diff vs the unsharded solve {worst:.2e}")


if __name__ == "__main__":
    main()
