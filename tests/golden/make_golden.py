"""Generate the golden fixtures from the REAL reference (oracle/_ref).

Run here (where /root/reference exists and `make ref` built
oracle/_ref/libjofc_ref.so):

    python tests/golden/make_golden.py

Writes tests/golden/golden.npz: inputs and reference outputs of every
hot-path entry point on small seeded cases.  tests/test_oracle.py replays
them against the C restatement (oracle/jofc_oracle.c) on any box, and the
GPU parity tests replay them against the CUDA path.  Inputs are drawn with
numpy's PCG64 (seeded) and the reference's own distance routine, so the
fixture, not the generator, is the source of truth.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.oracle import Reference, Spec  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")


def weight_family(m, w):
    """The three families of proj/tests/oracle_helpers.hpp:118-134 (restated)."""
    idx = np.arange(m)
    gen = np.where(idx[:, None] == idx[None, :], w * (1 + 0.1 * idx[:, None]),
                   w * (1 + 0.25 * np.abs(idx[:, None] - idx[None, :])))
    return [("uniform", Spec.uniform(w)), ("general", Spec.general_(gen)),
            ("product", Spec.product(w * (1 + 0.5 * idx), 1.5))]


def spec_arrays(prefix, spec, store):
    store[prefix + "kind"] = np.array({"uniform": 0, "general": 1, "product": 2}[spec.kind])
    store[prefix + "w"] = np.array(spec.w)
    store[prefix + "scale"] = np.array(spec.scale)
    if spec.general is not None:
        store[prefix + "general"] = spec.general
    if spec.within is not None:
        store[prefix + "within"] = spec.within


def main():
    R = Reference()
    rng = np.random.default_rng(20150312)
    store = {}
    cases = []

    # Rng stream pins (proj/include/jofc/rng.hpp)
    store["rng_u64_seed5"] = R.u64(5, 700)
    store["rng_normal_seed7"] = R.normals(7, 1001)

    # weights: W and W^-1 over the grid of proj/tests/test_weights.cpp:58-67
    wi = 0
    for m in (1, 2, 3, 5):
        for n in (2, 4, 7):
            for w in (0.1, 1.0, 10.0):
                for name, spec in weight_family(m, w):
                    p = f"w{wi}_"
                    spec_arrays(p, spec, store)
                    store[p + "mn"] = np.array([m, n])
                    store[p + "W"] = R.script_w(spec, m, n)
                    store[p + "Winv"] = R.script_w_inverse(spec, m, n)
                    wi += 1
    store["n_weights"] = np.array(wi)

    # in-sample: step / stress / 25-iteration solve on the grid of
    # proj/tests/test_embed_core.cpp:170-183 plus tile-boundary sizes.
    ci = 0
    for m in (1, 2, 3):
        for n in (3, 5, 8, 63, 65):
            for d in (1, 2, 3, 5):
                if n >= 63 and d not in (2, 5):
                    continue
                for name, spec in weight_family(m, [0.5, 1.0, 10.0][ci % 3]):
                    feats = [rng.normal(size=(n, 3)) * 2.0 for _ in range(m)]
                    delta = np.stack([R.distance_matrix(f) for f in feats])
                    x = rng.normal(size=(m, n, d))
                    p = f"c{ci}_"
                    spec_arrays(p, spec, store)
                    store[p + "delta"] = delta
                    store[p + "x"] = x
                    store[p + "stress"] = np.array(R.raw_stress(delta, spec, x))
                    store[p + "step"] = R.guttman_step_fast(delta, spec, x)
                    res = R.fjofc_embed(delta, spec, x, 1e-300, 25)
                    store[p + "solve_x"] = res.x
                    store[p + "solve_trace"] = res.trace
                    store[p + "solve_iters"] = np.array(res.iterations)
                    res2 = R.fjofc_embed(delta, spec, x, 1e-6, 200)
                    store[p + "eps_x"] = res2.x
                    store[p + "eps_trace"] = res2.trace
                    store[p + "eps_iters"] = np.array(res2.iterations)
                    R.release()
                    ci += 1
    store["n_cases"] = np.array(ci)

    # out-of-sample: step / stress / embed (proj/tests/test_oos.cpp:136-148 grid)
    oi = 0
    for m in (1, 2, 4):
        for n in (5, 9, 70):
            for d in (1, 2, 3):
                for w in (1.0, 10.0):
                    x = rng.normal(size=(m, n, d))
                    deltas = np.abs(rng.normal(size=(m, n))) + 0.1
                    y = rng.normal(size=(m, d)) * 1.5
                    p = f"o{oi}_"
                    store[p + "x"], store[p + "deltas"], store[p + "y"] = x, deltas, y
                    store[p + "w"] = np.array(w)
                    store[p + "stress"] = np.array(R.oos_stress(y, x, deltas, w))
                    store[p + "step"] = R.oos_step_fast(y, x, deltas, w)
                    e = R.oos_embed(x, deltas, w, 1e-6, 300, 11 + oi)
                    store[p + "seed"] = np.array(11 + oi)
                    store[p + "embed_y"] = e.x
                    store[p + "embed_trace"] = e.trace
                    store[p + "embed_iters"] = np.array(e.iterations)
                    oi += 1
    store["n_oos"] = np.array(oi)

    # edge cases: coincident rows (d == 0 guard), zero dissimilarity, n == 2
    delta = np.zeros((1, 3, 3))
    delta[0, 0, 1] = delta[0, 1, 0] = 1.0
    delta[0, 0, 2] = delta[0, 2, 0] = 2.0
    delta[0, 1, 2] = delta[0, 2, 1] = 1.5
    x = np.zeros((1, 3, 2))
    x[0, 2, 0] = 1.0
    store["edge_coincident_delta"], store["edge_coincident_x"] = delta, x
    store["edge_coincident_step"] = R.guttman_step_fast(delta, Spec.uniform(1.0), x)
    store["edge_coincident_stress"] = np.array(R.raw_stress(delta, Spec.uniform(1.0), x))
    R.release()
    z = np.zeros((2, 5, 5))
    xz = rng.normal(size=(2, 5, 2))
    store["edge_zero_x"] = xz
    store["edge_zero_step"] = R.guttman_step_fast(z, Spec.uniform(1.0), xz)
    store["edge_zero_stress"] = np.array(R.raw_stress(z, Spec.uniform(1.0), xz))
    R.release()

    np.savez_compressed(OUT, **store)
    print(f"wrote {OUT}: {len(store)} arrays, {ci} in-sample cases, {oi} oos cases, "
          f"{wi} weight cases")


if __name__ == "__main__":
    main()
