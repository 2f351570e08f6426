"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Tolerances (BASELINE.json north_star): final X within 1e-8 relative
Frobenius, stress within 1e-10 relative.  Single steps are held tighter
(1e-12), since only summation order and the rsqrt+Newton ratio differ.
"""
import numpy as np
import pytest

import paper_1502_03391_b200 as jg
from conftest import golden_spec, rel, rel_fro
from oracle.oracle import Port, Spec, best_available
from paper_1502_03391_b200 import workloads

pytestmark = pytest.mark.gpu

X_TOL = 1e-8
S_TOL = 1e-10
STEP_TOL = 1e-12
# Stress entries are compared at S_TOL relative; when a tiny-n case fits the
# data almost exactly (sigma_t ~ 1e-10 sigma_0) the relative error of such a
# near-zero sum is meaningless, so an absolute floor of 1e-13 sigma_0 applies
# (rounding of the individual residual terms is ~1e-16 of their scale).
ABS_FLOOR = 1e-13


def trace_close(got, ref):
    s0 = abs(ref[0])
    k = min(len(got), len(ref))
    return all(abs(a - b) <= S_TOL * abs(b) + ABS_FLOOR * s0 for a, b in zip(got[:k], ref[:k]))


@pytest.fixture(scope="module")
def dev():
    d = jg.Device(0)
    yield d
    d.close()


@pytest.fixture(scope="module")
def P():
    return Port()


def as_problem(delta):
    return jg.OmnibusProblem(list(delta), validate=False)


def test_golden_steps_and_stress(dev, golden):
    for i in range(int(golden["n_cases"])):
        p = f"c{i}_"
        spec = golden_spec(golden, p, "product")
        delta, x = golden[p + "delta"], golden[p + "x"]
        prob = as_problem(delta)
        s = jg.raw_stress(x, prob, spec, device=dev)
        assert rel(s, float(golden[p + "stress"])) < STEP_TOL, p
        step = jg.guttman_step_fast(x, prob, spec, device=dev)
        assert rel_fro(step, golden[p + "step"]) < STEP_TOL, p


def test_golden_solves(dev, golden):
    for i in range(int(golden["n_cases"])):
        p = f"c{i}_"
        spec = golden_spec(golden, p, "product")
        delta, x = golden[p + "delta"], golden[p + "x"]
        prob = as_problem(delta)
        opt = jg.SolveOptions(dim=x.shape[2], eps=1e-300, max_iterations=25,
                              init=jg.InitKind.provided, init_config=x)
        r = jg.fjofc_embed(prob, spec, opt, device=dev)
        ref_tr = golden[p + "solve_trace"]
        assert min(len(r.stress_trace), len(ref_tr)) >= 2
        assert trace_close(r.stress_trace, ref_tr), p
        if r.iterations == int(golden[p + "solve_iters"]):
            assert rel_fro(r.config, golden[p + "solve_x"]) < X_TOL, p


def test_eps_termination_matches(dev, golden):
    agree = 0
    total = 0
    for i in range(int(golden["n_cases"])):
        p = f"c{i}_"
        spec = golden_spec(golden, p, "product")
        delta, x = golden[p + "delta"], golden[p + "x"]
        opt = jg.SolveOptions(dim=x.shape[2], eps=1e-6, max_iterations=200,
                              init=jg.InitKind.provided, init_config=x)
        r = jg.fjofc_embed(as_problem(delta), spec, opt, device=dev)
        total += 1
        if r.iterations == int(golden[p + "eps_iters"]):
            agree += 1
            assert rel_fro(r.config, golden[p + "eps_x"]) < X_TOL, p
    # the stop index may flip only when a decrease sits exactly at eps
    assert agree >= total - 2, (agree, total)


@pytest.mark.parametrize("d", list(range(1, 11)))
def test_every_dim_and_tile_boundary(dev, P, d):
    rng = np.random.default_rng(100 + d)
    for m, n in ((1, 2), (2, 3), (3, 64), (2, 65), (1, 127), (2, 130), (3, 200)):
        delta = np.stack([P.distance_matrix(rng.normal(size=(n, 3)) * 2) for _ in range(m)])
        x = rng.normal(size=(m, n, d))
        for spec_o, spec in ((Spec.uniform(0.7), jg.WeightSpec.uniform(0.7)),
                             (Spec.product(np.linspace(0.5, 1.5, m), 1.3),
                              jg.WeightSpec.product(np.linspace(0.5, 1.5, m), 1.3))):
            prob = as_problem(delta)
            assert rel(jg.raw_stress(x, prob, spec, device=dev),
                       P.raw_stress(delta, spec_o, x)) < STEP_TOL
            assert rel_fro(jg.guttman_step_fast(x, prob, spec, device=dev),
                           P.guttman_step_fast(delta, spec_o, x)) < STEP_TOL, (m, n, d)


def test_coincident_rows_guard(dev, golden):
    u = jg.WeightSpec.uniform(1.0)
    prob = as_problem(golden["edge_coincident_delta"])
    x = golden["edge_coincident_x"]
    step = jg.guttman_step_fast(x, prob, u, device=dev)
    assert rel_fro(step, golden["edge_coincident_step"]) < STEP_TOL
    assert rel(jg.raw_stress(x, prob, u, device=dev),
               float(golden["edge_coincident_stress"])) < STEP_TOL


def test_zero_dissimilarity(dev, golden):
    u = jg.WeightSpec.uniform(1.0)
    prob = as_problem(np.zeros((2, 5, 5)))
    x = golden["edge_zero_x"]
    step = jg.guttman_step_fast(x, prob, u, device=dev)
    assert np.array_equal(step, golden["edge_zero_step"])
    assert rel(jg.raw_stress(x, prob, u, device=dev), float(golden["edge_zero_stress"])) < 1e-13


def test_nan_init_raises_numerical_error(dev, P):
    rng = np.random.default_rng(48)
    delta = np.stack([P.distance_matrix(rng.normal(size=(5, 2))) for _ in range(2)])
    x = rng.normal(size=(2, 5, 2))
    x[0, 0, 0] = np.nan
    opt = jg.SolveOptions(dim=2, init=jg.InitKind.provided, init_config=x)
    with pytest.raises(jg.NumericalError, match="initial configuration"):
        jg.fjofc_embed(as_problem(delta), jg.WeightSpec.uniform(1.0), opt, device=dev)


def test_shape_errors(dev, P):
    rng = np.random.default_rng(50)
    delta = np.stack([P.distance_matrix(rng.normal(size=(5, 2))) for _ in range(2)])
    wrong = rng.normal(size=(2, 6, 2))
    with pytest.raises(jg.InvalidArgument):
        jg.raw_stress(wrong, as_problem(delta), jg.WeightSpec.uniform(1.0), device=dev)
    with pytest.raises(jg.InvalidArgument):
        jg.guttman_step_fast(wrong, as_problem(delta), jg.WeightSpec.uniform(1.0), device=dev)
    bad = delta.copy()
    bad[0, 0, 1] = -1.0
    with pytest.raises(jg.InvalidArgument):
        dev.upload(as_problem(bad))


def test_realizable_data_converges_immediately(dev, P):
    # proj/tests/test_embed_core.cpp:277-292
    rng = np.random.default_rng(45)
    x = rng.normal(size=(10, 2))
    x -= x.mean(axis=0)
    delta = P.distance_matrix(x)
    opt = jg.SolveOptions(dim=2, init=jg.InitKind.provided, init_config=np.stack([x] * 3))
    r = jg.fjofc_embed(as_problem(np.stack([delta] * 3)), jg.WeightSpec.uniform(1.0), opt,
                       device=dev)
    assert r.iterations <= 2
    assert r.final_stress() < 1e-16
    assert r.terminated == jg.Termination.converged


def test_normalize_option(dev, P):
    rng = np.random.default_rng(49)
    delta = np.stack([P.distance_matrix(rng.normal(size=(30, 2)) * 3) for _ in range(2)])
    x = rng.normal(size=(2, 30, 2))
    opt = jg.SolveOptions(dim=2, eps=1e-300, max_iterations=20, init=jg.InitKind.provided,
                          init_config=x, normalize=True)
    r = jg.fjofc_embed(as_problem(delta), jg.WeightSpec.uniform(1.0), opt, device=dev)
    ref = P.fjofc_embed(delta, Spec.uniform(1.0), x, 1e-300, 20, normalize=True)
    assert rel_fro(r.config, ref.x) < X_TOL
    assert max(rel(a, b) for a, b in zip(r.stress_trace, ref.trace)) < S_TOL


def test_features_upload_is_bitwise_dense_upload(dev, P):
    wl = workloads.make(3, n=300)
    x = wl.x0()
    spec = wl.spec
    dev.upload_features(wl.in_features)
    a = dev.lib  # noqa: F841
    import ctypes as C
    from paper_1502_03391_b200._capi import dptr
    s1 = C.c_double()
    jg._capi.check(dev.lib.jofc_raw_stress(dev.h, C.byref(spec.c()), wl.d, dptr(x), C.byref(s1)))
    dev._problem_key = None
    s2 = jg.raw_stress(x, as_problem(wl.dense_delta()), spec, device=dev)
    assert s1.value == s2  # same packed bits, same kernel, same order


# ------------------------------------------------------------------ configs
def _config_parity(dev, P, cfg, n=None, iters=None):
    """Full solve vs the reference (oracle/_ref, OpenMP) or the port."""
    wl = workloads.make(cfg, n=n)
    iters = iters or wl.iterations
    delta = wl.dense_delta()
    x0 = wl.x0()
    spec_o = (Spec.general_(wl.spec.general) if wl.general_weights else Spec.uniform(wl.w))
    R = best_available()
    ref = R.fjofc_embed(delta, spec_o, x0, 1e-300, iters, parallel=True)
    opt = jg.SolveOptions(dim=wl.d, eps=1e-300, max_iterations=iters,
                          init=jg.InitKind.provided, init_config=x0)
    r = jg.fjofc_embed(as_problem(delta), wl.spec, opt, device=dev)
    k = min(len(r.stress_trace), len(ref.trace))
    worst = max(rel(a, b) for a, b in zip(r.stress_trace[:k], ref.trace[:k]))
    assert worst < S_TOL, worst
    assert r.iterations == ref.iterations, (r.iterations, ref.iterations)
    assert rel_fro(r.config, ref.x) < X_TOL
    return r


def test_config1_full(dev, P):
    _config_parity(dev, P, 1)


def test_config2_full(dev, P):
    _config_parity(dev, P, 2)


def test_config5_in_sample_full(dev, P):
    _config_parity(dev, P, 5)


def test_config4_reduced(dev, P):
    _config_parity(dev, P, 4, n=1500, iters=30)


def test_config3_reduced(dev, P):
    _config_parity(dev, P, 3, n=2500, iters=20)


# Full BASELINE sizes and iteration counts (C3: 2 x 20000^2, C4: 10 x 10000^2
# dense host Delta, 100 iterations) against the reference library itself
# (oracle/_ref, OpenMP on the host cores): every stress-trace entry, the
# iteration count and the final X.  Then the bench's path (Delta built on the
# device from the features, bit-identical) reproduces that solve.
@pytest.mark.parametrize("cfg", [3, 4])
def test_full_size_against_reference(dev, P, cfg):
    r = _config_parity(dev, P, cfg)
    wl = workloads.make(cfg)
    assert r.iterations == wl.iterations
    tr = r.stress_trace
    assert all(b < a for a, b in zip(tr, tr[1:]))  # strict decrease: the stop rule never fired
    opt = jg.SolveOptions(dim=wl.d, eps=1e-300, max_iterations=wl.iterations,
                          init=jg.InitKind.provided, init_config=wl.x0())
    prob = dev.upload_features(wl.in_features)
    again = jg.fjofc_embed(prob, wl.spec, opt, device=dev)
    assert again.iterations == r.iterations
    assert max(rel(a, b) for a, b in zip(again.stress_trace, tr)) < 1e-12
    assert rel_fro(again.config, r.config) < 1e-12


# ------------------------------------------------------------------ out-of-sample
def test_oos_golden(dev, golden):
    for i in range(int(golden["n_oos"])):
        p = f"o{i}_"
        x, dl, y, w = golden[p + "x"], golden[p + "deltas"], golden[p + "y"], float(golden[p + "w"])
        assert rel(jg.oos_stress(y, x, dl, w, device=dev), float(golden[p + "stress"])) < STEP_TOL
        assert rel_fro(jg.oos_step_fast(y, x, dl, w, device=dev), golden[p + "step"]) < STEP_TOL
        e = jg.oos_embed(x, dl, w, jg.OosOptions(1e-6, 300), int(golden[p + "seed"]), device=dev)
        assert trace_close(e.stress_trace, golden[p + "embed_trace"]), p
        assert rel_fro(e.y, golden[p + "embed_y"]) < 1e-7, p


@pytest.mark.parametrize("n,d", [(333, 10), (1031, 7), (517, 1), (2049, 3)])
def test_oos_batch_odd_sizes_and_dims(dev, P, n, d):
    # odd n and odd d: X chunks start off 16-byte boundaries (TMA staging), the
    # widest d uses the > 48 KB shared-memory launch
    rng = np.random.default_rng(n + d)
    m, k = 2, 21
    x = rng.normal(size=(m, n, d))
    yt = rng.normal(size=(k, m, d))
    od = np.stack([[np.sqrt(((x[l] - yt[q, l]) ** 2).sum(1)) + 0.05 * rng.random(n)
                    for l in range(m)] for q in range(k)])
    y0 = np.stack([jg.oos_start(x, 77 + q) for q in range(k)])
    y, tr, its = jg.oos_embed_batch(x, od, 0.7, y0, jg.OosOptions(1e-300, 40),
                                    fixed_iterations=True, device=dev)
    yr, trr, itr = P.oos_batch(x, od, 0.7, y0, 1e-300, 40, fixed=True)
    for q in range(k):
        assert rel_fro(y[q], yr[q]) < X_TOL
        assert np.max(np.abs(tr[q] - trr[q]) / np.abs(trr[q])) < S_TOL


def test_oos_batch_config5(dev, P):
    wl = workloads.make(5, n=1200)
    x = P.fjofc_embed(wl.dense_delta(), Spec.uniform(wl.w), wl.x0(), 1e-300, 30).x
    od = wl.oos_deltas()[:200]
    y0 = np.stack([jg.oos_start(x, workloads.OOS_SEED + q) for q in range(200)])
    y, tr, its = jg.oos_embed_batch(x, od, wl.w, y0, jg.OosOptions(1e-300, 100),
                                    fixed_iterations=True, device=dev)
    yr, trr, itr = P.oos_batch(x, od, wl.w, y0, 1e-300, 100, fixed=True)
    assert np.all(its == 100) and np.all(itr == 100)
    for q in range(200):
        assert rel_fro(y[q], yr[q]) < X_TOL
        assert np.max(np.abs(tr[q] - trr[q]) / np.abs(trr[q])) < S_TOL


def test_maximum_size_realizable_fixed_point(dev):
    # n = 100000 (n^2 > 2^32, 40 GB of packed Delta built on the device from the
    # features): for realizable data the configuration that generated Delta
    # has zero fidelity and is a fixed point of the transform
    # (B(X*) X* = n X* for centred X*; proj/tests/test_embed_core.cpp:277-292
    # at maximum size)
    rng = np.random.default_rng(77)
    n, d = 100_000, 3
    xs = rng.normal(size=(n, d)) * 10.0
    xs -= xs.mean(axis=0)
    prob = dev.upload_features(xs[None])
    assert dev.problem_pairs() == n * (n - 1) / 2
    u = jg.WeightSpec.uniform(1.0)
    x = xs[None].copy()
    scale = float(np.sum(xs * xs)) * n  # ~ sum of delta^2 over the pairs
    assert jg.raw_stress(x, prob, u, device=dev) < 1e-24 * scale
    step = jg.guttman_step_fast(x, prob, u, device=dev)
    assert rel_fro(step, x) < 1e-13


def test_maximum_size_oos_fixed_points(dev):
    # out of sample at n = 200000 in-sample objects, m = 3, a batch of 64
    # points: a point whose dissimilarities are its true distances to every
    # modality's configuration (the same location in each) is a fixed point of
    # the update (r_k = 1: psi = n, xi = 0) with zero stress
    rng = np.random.default_rng(78)
    m, n, d, k = 3, 200_000, 2, 64
    x = rng.normal(size=(m, n, d)) * 5.0
    ys = rng.normal(size=(k, d)) * 5.0
    deltas = np.sqrt(((x[None, :, :, :] - ys[:, None, None, :]) ** 2).sum(-1))  # k x m x n
    y0 = np.repeat(ys[:, None, :], m, axis=1)
    y, traces, its = jg.oos_embed_batch(x, deltas, 0.5, y0, jg.OosOptions(eps=1e-300,
                                                                          max_iterations=3),
                                        fixed_iterations=True, device=dev)
    assert np.all(its == 3)
    assert np.max(np.abs(y - y0)) < 1e-12 * np.max(np.abs(y0))
    assert np.all(traces[:, :4] < 1e-20 * n * 25.0)
    assert jg.oos_stress(y0[0], x, deltas[0], 0.5, device=dev) < 1e-20 * n * 25.0
    assert np.max(np.abs(jg.oos_step_fast(y0[5], x, deltas[5], 0.5, device=dev) - y0[5])) < 1e-12 * 5


def test_many_modalities(dev, P):
    # m = 16 modalities (the epilogue's m x m mix and m(m-1)/2 commensurability
    # pairs, product weights) against the port, steps and a short solve
    rng = np.random.default_rng(66)
    m, n, d = 16, 150, 3
    z = rng.normal(size=(n, 3))
    delta = np.stack([P.distance_matrix(z + 0.3 * rng.normal(size=(n, 3))) for _ in range(m)])
    x = rng.normal(size=(m, n, d))
    within = np.linspace(0.5, 2.0, m)
    spec_o, spec = Spec.product(within, 0.8), jg.WeightSpec.product(within, 0.8)
    prob = as_problem(delta)
    assert rel(jg.raw_stress(x, prob, spec, device=dev), P.raw_stress(delta, spec_o, x)) < STEP_TOL
    assert rel_fro(jg.guttman_step_fast(x, prob, spec, device=dev),
                   P.guttman_step_fast(delta, spec_o, x)) < STEP_TOL
    opt = jg.SolveOptions(dim=d, eps=1e-300, max_iterations=30, init=jg.InitKind.provided,
                          init_config=x)
    r = jg.fjofc_embed(prob, spec, opt, device=dev)
    ref = P.fjofc_embed(delta, spec_o, x, 1e-300, 30)
    assert r.iterations == ref.iterations
    assert rel_fro(r.config, ref.x) < X_TOL
    assert trace_close(r.stress_trace, ref.trace)


def test_oos_batch_many_modalities_with_stop_rule(dev, P):
    # m = 7 views per point and the per-point stop rule (not a fixed count):
    # each point's iterations, y and trace against the port
    rng = np.random.default_rng(71)
    m, n, d, k = 7, 300, 4, 37
    x = rng.normal(size=(m, n, d))
    yt = rng.normal(size=(k, m, d))
    od = np.stack([[np.sqrt(((x[l] - yt[q, l]) ** 2).sum(1)) + 0.05 * rng.random(n)
                    for l in range(m)] for q in range(k)])
    y0 = np.stack([jg.oos_start(x, 500 + q) for q in range(k)])
    y, tr, its = jg.oos_embed_batch(x, od, 0.4, y0, jg.OosOptions(1e-7, 200), device=dev)
    yr, trr, itr = P.oos_batch(x, od, 0.4, y0, 1e-7, 200)
    agree = 0
    for q in range(k):
        if its[q] == itr[q]:
            agree += 1
            assert rel_fro(y[q], yr[q]) < X_TOL
            assert np.max(np.abs(tr[q][: its[q] + 1] - trr[q][: its[q] + 1])
                          / np.abs(trr[q][: its[q] + 1])) < S_TOL
    assert agree >= k - 1, (agree, k)  # a stop may flip only at a decrease sitting at eps
