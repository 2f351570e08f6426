"""One-off randomised sweep of the large-n in-sample route (per-launch graph, identity-form
fidelity, many bands / CTAs) over every embedding dimension, against the reference itself
(oracle/_ref, OpenMP) -- the suite's own sweep (tests/test_gpu_fuzz.py) stops at n = 2300,
the full-size parity tests cover d = 3 and d = 5 only.

python scripts/fuzz_large.py [seed [cases]]     (needs a GPU and oracle/_ref)
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import paper_1502_03391_b200 as jg  # noqa: E402
from oracle.oracle import Reference, Spec  # noqa: E402  (the checker)


def rel_fro(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(b))


def main():
    seed = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    cases = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    R = Reference()
    dev = jg.Device(0)
    worst_x = worst_s = 0.0
    for case in range(cases):
        rng = np.random.default_rng(seed * 1000 + case)
        d = case % 10 + 1                      # every d = 1..10 in turn
        m = int(rng.integers(1, 4))
        n = int(rng.choice([2301, 3000, 4095, 4096, 4097, 5555, 6400, 8191, 8200]))
        its = int(rng.integers(2, 7))
        p = max(d, 3)
        z = rng.normal(size=(n, p))
        feats = np.stack([z + 0.2 * rng.normal(size=(n, p)) for _ in range(m)])
        delta = np.stack([R.distance_matrix(f, parallel=True) for f in feats])
        if rng.random() < 0.5:                 # a duplicated object (dist == 0 guard)
            i, j = (int(v) for v in rng.integers(0, n, size=2))
            if i != j:
                delta[:, i, :] = delta[:, j, :]
                delta[:, :, i] = delta[:, :, j]
                delta[:, i, i] = 0.0
                delta[:, i, j] = delta[:, j, i] = 0.0
        kind = int(rng.integers(0, 2))
        if kind == 0:
            w = float(rng.uniform(0.1, 2.0))
            spec, sref = jg.WeightSpec.uniform(w), Spec.uniform(w)
        else:
            a = rng.uniform(0.2, 1.0, size=(m, m))
            a = 0.5 * (a + a.T)
            spec, sref = jg.WeightSpec.general(a), Spec.general_(a)
        x0 = rng.normal(size=(m, n, d))
        if rng.random() < 0.5:
            x0[:, 1, :] = x0[:, 0, :]          # coincident start rows
        t0 = time.perf_counter()
        opt = jg.SolveOptions(dim=d, eps=1e-300, max_iterations=its, init=jg.InitKind.provided,
                              init_config=x0)
        r = jg.fjofc_embed(jg.OmnibusProblem(list(delta)), spec, opt, device=dev)
        ref = R.fjofc_embed(delta, sref, x0, 1e-300, its, parallel=True)
        ex = rel_fro(r.config, ref.x)
        es = max(abs(a_ - b_) / abs(b_) for a_, b_ in zip(r.stress_trace, ref.trace))
        worst_x, worst_s = max(worst_x, ex), max(worst_s, es)
        ok = r.iterations == ref.iterations and ex < 1e-8 and es < 1e-10
        print(f"case {case}: m={m} n={n} d={d} its={its} kind={kind} X {ex:.2e} trace {es:.2e} "
              f"{'ok' if ok else 'MISMATCH'} ({time.perf_counter() - t0:.1f} s)", flush=True)
        if not ok:
            sys.exit(1)
    print(f"all {cases} cases ok: worst X rel err {worst_x:.2e}, worst trace rel err {worst_s:.2e}")
    dev.close()


if __name__ == "__main__":
    main()
