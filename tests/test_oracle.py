"""The CPU oracle (oracle/jofc_oracle.c) pinned against the real reference.

* golden fixtures written by tests/golden/make_golden.py from oracle/_ref
  (the unmodified reference sources) are replayed bit-for-bit;
* known-answer pins of proj/tests/test_weights.cpp:12-56;
* when oracle/_ref is present, live random cases compare both directly.
"""
import os

import numpy as np
import pytest

from conftest import golden_spec
from oracle.oracle import REF_SO, InvalidArgument, NumericalError, Port, Reference, Spec

P = Port()


def test_rng_stream_matches_reference(golden):
    assert np.array_equal(P.u64(5, 700), golden["rng_u64_seed5"])
    assert np.array_equal(P.normals(7, 1001), golden["rng_normal_seed7"])


def test_weights_known_answers():
    # proj/tests/test_weights.cpp:12-56
    w = P.script_w(Spec.uniform(1.0), 2, 3)
    assert np.allclose(w, [[4, -1], [-1, 4]])
    assert np.allclose(P.script_w(Spec.uniform(1.0), 1, 5), [[5.0]])
    assert np.allclose(P.script_w(Spec.product([1.0, 2.0], 1.0), 2, 3), [[5, -2], [-2, 8]])
    inv = P.script_w_inverse(Spec.uniform(1.0), 2, 3)
    assert np.allclose(inv, [[4 / 15, 1 / 15], [1 / 15, 4 / 15]], rtol=1e-15)
    assert np.isclose(P.script_w_inverse(Spec.uniform(1.0), 1, 5)[0, 0], 0.2)
    inv = P.script_w_inverse(Spec.product([1.0, 1.0], 1.0), 2, 4)
    assert np.isclose(inv[0, 0], 5 / 24) and np.isclose(inv[0, 1], 1 / 24)
    for bad in (0.0, -1.0):
        with pytest.raises(InvalidArgument):
            P.script_w(Spec.uniform(bad), 2, 3)


def test_weights_golden(golden):
    for i in range(int(golden["n_weights"])):
        p = f"w{i}_"
        m, n = (int(v) for v in golden[p + "mn"])
        spec = golden_spec(golden, p)
        assert np.array_equal(P.script_w(spec, m, n), golden[p + "W"])
        assert np.array_equal(P.script_w_inverse(spec, m, n), golden[p + "Winv"])


def test_in_sample_golden_bit_exact(golden):
    for i in range(int(golden["n_cases"])):
        p = f"c{i}_"
        spec = golden_spec(golden, p)
        delta, x = golden[p + "delta"], golden[p + "x"]
        assert P.raw_stress(delta, spec, x) == float(golden[p + "stress"]), p
        assert np.array_equal(P.guttman_step_fast(delta, spec, x), golden[p + "step"]), p
        r = P.fjofc_embed(delta, spec, x, 1e-300, 25)
        assert r.iterations == int(golden[p + "solve_iters"])
        assert np.array_equal(r.x, golden[p + "solve_x"]) and np.array_equal(
            r.trace, golden[p + "solve_trace"]), p
        r = P.fjofc_embed(delta, spec, x, 1e-6, 200)
        assert r.iterations == int(golden[p + "eps_iters"]), p
        assert np.array_equal(r.x, golden[p + "eps_x"]), p


def test_oos_golden_bit_exact(golden):
    for i in range(int(golden["n_oos"])):
        p = f"o{i}_"
        x, dl, y, w = golden[p + "x"], golden[p + "deltas"], golden[p + "y"], float(golden[p + "w"])
        assert P.oos_stress(y, x, dl, w) == float(golden[p + "stress"])
        assert np.array_equal(P.oos_step_fast(y, x, dl, w), golden[p + "step"])
        e = P.oos_embed(x, dl, w, 1e-6, 300, int(golden[p + "seed"]))
        assert e.iterations == int(golden[p + "embed_iters"])
        assert np.array_equal(e.x, golden[p + "embed_y"])
        assert np.array_equal(e.trace, golden[p + "embed_trace"])


def test_edge_cases_golden(golden):
    u = Spec.uniform(1.0)
    d, x = golden["edge_coincident_delta"], golden["edge_coincident_x"]
    assert np.array_equal(P.guttman_step_fast(d, u, x), golden["edge_coincident_step"])
    assert P.raw_stress(d, u, x) == float(golden["edge_coincident_stress"])
    z = np.zeros((2, 5, 5))
    assert np.array_equal(P.guttman_step_fast(z, u, golden["edge_zero_x"]), golden["edge_zero_step"])


def test_numerical_errors():
    rng = np.random.default_rng(1)
    f = rng.normal(size=(5, 2))
    d = np.stack([P.distance_matrix(f)] * 2)
    x = rng.normal(size=(2, 5, 2))
    x[0, 0, 0] = np.nan
    with pytest.raises(NumericalError, match="initial configuration"):
        P.fjofc_embed(d, Spec.uniform(1.0), x, 1e-6, 10)


@pytest.mark.skipif(not os.path.exists(REF_SO), reason="oracle/_ref not built here")
def test_live_reference_random_cases():
    R = Reference()
    rng = np.random.default_rng(7)
    for m in (1, 2, 4):
        for n in (2, 17, 40):
            d = int(rng.integers(1, 6))
            feats = [rng.normal(size=(n, 4)) for _ in range(m)]
            delta = np.stack([R.distance_matrix(f) for f in feats])
            assert np.array_equal(delta, np.stack([P.distance_matrix(f) for f in feats]))
            x = rng.normal(size=(m, n, d))
            spec = Spec.uniform(float(rng.uniform(0.1, 3)))
            a = P.fjofc_embed(delta, spec, x, 1e-300, 40)
            b = R.fjofc_embed(delta, spec, x, 1e-300, 40)
            assert a.iterations == b.iterations
            assert np.array_equal(a.x, b.x) and np.array_equal(a.trace, b.trace)
            R.release()
