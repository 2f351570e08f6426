"""Delta asymmetric within the reference's tolerance (OmnibusProblem accepts
|Delta_ij - Delta_ji| <= 1e-9 max(1, max|Delta|), proj/src/problem.cpp:21-23).

The reference's step reads BOTH triangles (row i uses Delta(i, k),
proj/src/solver.cpp:45) while its stress reads the upper one
(proj/src/stress.cpp:46-59); the device keeps the packed upper triangle only.
So: the stress is exact (same entries), and the step differs from the
reference's by at most the asymmetry itself -- a documented deviation
 that keeps the X tolerance (1e-8)."""
import os

import numpy as np
import pytest

import paper_1502_03391_b200 as jg
from conftest import rel, rel_fro
from oracle.oracle import REF_SO, Spec

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not os.path.exists(REF_SO), reason="oracle/_ref not built")]


def asymmetric_problem(n=400, m=2, seed=4):
    from oracle.oracle import Port
    P = Port()
    rng = np.random.default_rng(seed)
    z = rng.normal(size=(n, 3))
    out = []
    for _ in range(m):
        d = P.distance_matrix(z + 0.1 * rng.normal(size=(n, 3)))
        scale = max(1.0, float(np.max(np.abs(d))))
        e = rng.uniform(-1.0, 1.0, size=(n, n)) * 0.45e-9 * scale
        e = 0.5 * (e - e.T)  # antisymmetric: |Delta_ij - Delta_ji| = 2|e_ij| <= 0.9e-9 scale
        out.append(np.abs(d + e) * (1 - np.eye(n)))
    return np.stack(out)


def test_asymmetric_delta_within_tolerance():
    from oracle.oracle import Reference
    R = Reference()
    delta = asymmetric_problem()
    m, n, _ = delta.shape
    asym = max(float(np.max(np.abs(d - d.T))) for d in delta)
    assert 0 < asym <= 1e-9 * max(1.0, float(np.max(delta)))
    prob = jg.OmnibusProblem(list(delta))  # the reference's validation accepts it
    spec, spec_o = jg.WeightSpec.uniform(0.5), Spec.uniform(0.5)
    x = np.random.default_rng(1).normal(size=(m, n, 3))
    # stress: the same upper-triangle entries -> agreement to rounding
    assert rel(jg.raw_stress(x, prob, spec), R.raw_stress(delta, spec_o, x)) < 1e-12
    # step: bounded by the asymmetry (relative ~1e-9), not by rounding
    step_err = rel_fro(jg.guttman_step_fast(x, prob, spec), R.guttman_step_fast(delta, spec_o, x))
    assert step_err < 5e-9, step_err
    # a 30-iteration solve stays within the north-star X tolerance
    opt = jg.SolveOptions(dim=3, eps=1e-300, max_iterations=30, init=jg.InitKind.provided,
                          init_config=x)
    got = jg.fjofc_embed(prob, spec, opt)
    ref = R.fjofc_embed(delta, spec_o, x, 1e-300, 30)
    x_err = rel_fro(got.config, ref.x)
    s_err = max(rel(a, b) for a, b in zip(got.stress_trace, ref.trace))
    print(f"asymmetry {asym:.2e}: step rel err {step_err:.2e}, 30-it X rel err {x_err:.2e}, "
          f"max trace rel err {s_err:.2e}")
    assert got.iterations == ref.iterations and x_err < 1e-8
