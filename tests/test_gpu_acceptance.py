"""The reference's release gates that concern the hot path
(proj/tests/acceptance/acceptance_main.cpp, criteria 2, 3, 4 and 8; SURVEY.md
8c), restated as tests of THIS implementation: the GPU transforms against the
reference's dense Algorithm-1 transforms, the majorization and centring
properties of GPU solves, the GPU stress against the analytic gradient, and
the out-of-sample residual of a held-out object."""
import os

import numpy as np
import pytest

import paper_1502_03391_b200 as jg
from oracle.oracle import REF_SO, Spec

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not os.path.exists(REF_SO), reason="oracle/_ref not built")]


@pytest.fixture(scope="module")
def R():
    from oracle.oracle import Reference
    return Reference()


@pytest.fixture(scope="module")
def dev():
    return jg.Device(0)


def edm(x):
    diff = x[:, None, :] - x[None, :, :]
    return np.sqrt((diff * diff).sum(-1))


def random_problem(rng, n, m, d):
    return np.stack([edm(2.0 * rng.normal(size=(n, d))) for _ in range(m)])


def families(m, w):
    """(ours, reference) pairs of the three weight families."""
    g = np.array([[w * (1.0 + 0.1 * i) if i == j else w * (1.0 + 0.25 * abs(i - j))
                   for j in range(m)] for i in range(m)])
    within = [w * (1.0 + 0.5 * i) for i in range(m)]
    return [(jg.WeightSpec.uniform(w), Spec.uniform(w)),
            (jg.WeightSpec.general(g), Spec.general_(g)),
            (jg.WeightSpec.product(within, 1.5), Spec.product(within, 1.5))]


def test_gate2_step_equivalence_with_dense_reference(R, dev):
    # criterion 2: fast transform vs the dense L+ B X transform, max-abs < 1e-8
    rng = np.random.default_rng(202)
    worst = 0.0
    for m in (1, 2, 3):
        for n in (3, 5, 8):
            for d in (1, 2, 3):
                for w in (0.5, 1.0, 10.0):
                    for ours, ref in families(m, w):
                        delta = random_problem(rng, n, m, d)
                        x = rng.normal(size=(m, n, d))
                        prob = jg.OmnibusProblem(list(delta), validate=False)
                        got = jg.guttman_step_fast(x, prob, ours, device=dev)
                        want = R.guttman_step_reference(delta, ref, x)
                        worst = max(worst, float(np.max(np.abs(got - want))))
    assert worst < 1e-8, worst
    worst_oos = 0.0
    for m in (1, 2, 4):
        for n in (5, 9):
            for d in (1, 2):
                for w in (1.0, 10.0):
                    x = rng.normal(size=(m, n, d))
                    deltas = np.abs(rng.normal(size=(m, n))) + 0.1
                    y = 1.5 * rng.normal(size=(m, d))
                    got = jg.oos_step_fast(y, x, deltas, w, device=dev)
                    want = R.oos_step_reference(y, x, deltas, w)
                    worst_oos = max(worst_oos, float(np.max(np.abs(got - want))))
    assert worst_oos < 1e-8, worst_oos


def test_gate3_majorization_and_centring(dev):
    # criterion 3: 200 solves from the GPU initialisers; the stress never rises
    # (slack 1e-9) and every iterate is column-centred (1e-9)
    rng = np.random.default_rng(303)
    worst_rise, worst_mean = -np.inf, 0.0
    for inst in range(200):
        m, n, d = 1 + rng.integers(3), 4 + rng.integers(8), 1 + rng.integers(3)
        prob = jg.OmnibusProblem(list(random_problem(rng, n, m, d)), validate=False)
        spec = jg.WeightSpec.uniform(0.25 + 4.0 * rng.uniform())
        opt = jg.SolveOptions(dim=int(d), max_iterations=25, keep_config_trace=True,
                              init=jg.InitKind.averaged_procrustes if inst % 2 == 0
                              else jg.InitKind.imputed_cmds)
        r = jg.fjofc_embed(prob, spec, opt, device=dev)
        tr = r.stress_trace
        worst_rise = max([worst_rise] + [b - a for a, b in zip(tr, tr[1:])])
        for cfg in r.config_trace[1:]:
            worst_mean = max(worst_mean, float(np.max(np.abs(cfg.mean(axis=1)))))
    assert worst_rise <= 1e-9, worst_rise
    assert worst_mean < 1e-9, worst_mean


def test_gate4_stress_gradient(dev):
    # criterion 4: central differences of the GPU raw stress / oos stress
    # against the analytic gradients (relative gap < 1e-4)
    rng = np.random.default_rng(404)
    h = 1e-5
    worst = 0.0
    for _ in range(20):
        m, n, d = 1 + rng.integers(3), 4 + rng.integers(4), 1 + rng.integers(2)
        delta = random_problem(rng, n, m, d)
        prob = jg.OmnibusProblem(list(delta), validate=False)
        x = 2.0 * rng.normal(size=(m, n, d))
        w = 0.5 + rng.uniform()
        spec = jg.WeightSpec.uniform(w)
        # sigma = sum_l sum_{i<j} (delta - d)^2 + w sum_{l<l'} sum_k |x_k^l - x_k^l'|^2
        grad = np.zeros_like(x)
        for l in range(m):
            diff = x[l][:, None, :] - x[l][None, :, :]
            dist = np.sqrt((diff * diff).sum(-1))
            with np.errstate(divide="ignore", invalid="ignore"):
                coef = np.where(dist > 0, (dist - delta[l]) / dist, 0.0)
            grad[l] += 2.0 * (coef[:, :, None] * diff).sum(1)
            for l2 in range(m):
                if l2 != l:
                    grad[l] += 2.0 * w * (x[l] - x[l2])
        fd = np.zeros_like(x)
        for idx in np.ndindex(*x.shape):
            keep = x[idx]
            x[idx] = keep + h
            up = jg.raw_stress(x, prob, spec, device=dev)
            x[idx] = keep - h
            down = jg.raw_stress(x, prob, spec, device=dev)
            x[idx] = keep
            fd[idx] = (up - down) / (2.0 * h)
        worst = max(worst, float(np.linalg.norm(grad - fd) / np.linalg.norm(grad)))
    assert worst < 1e-4, worst
    worst_oos = 0.0
    for _ in range(20):
        m, n, d = 2 + rng.integers(3), 4 + rng.integers(5), 1 + rng.integers(2)
        w = 0.5 + rng.uniform()
        x = rng.normal(size=(m, n, d))
        deltas = np.abs(rng.normal(size=(m, n))) + 0.1
        y = 1.5 * rng.normal(size=(m, d))
        l22 = np.full((m, m), -w) + np.eye(m) * (n + m * w)
        grad = 2.0 * l22 @ (y - jg.oos_step_fast(y, x, deltas, w, device=dev))
        fd = np.zeros_like(y)
        for idx in np.ndindex(*y.shape):
            keep = y[idx]
            y[idx] = keep + h
            up = jg.oos_stress(y, x, deltas, w, device=dev)
            y[idx] = keep - h
            down = jg.oos_stress(y, x, deltas, w, device=dev)
            y[idx] = keep
            fd[idx] = (up - down) / (2.0 * h)
        worst_oos = max(worst_oos, float(np.linalg.norm(grad - fd) / np.linalg.norm(grad)))
    assert worst_oos < 1e-4, worst_oos


def test_gate8_out_of_sample_residual(R, dev):
    # criterion 8 (residual part): hold out the last of n = 200 objects (m = 10,
    # 3-d matched setting), embed the rest from the full solution restricted,
    # then place the held-out object out of sample; mean residual <= 0.3
    m, dim, n = 10, 3, 200
    total = 0.0
    for seed in range(1, 6):
        delta = R.generate_matched(n, m, dim, seed)
        full = jg.OmnibusProblem(list(delta), validate=False)
        spec = jg.WeightSpec.uniform(1.0)
        fr = jg.fjofc_embed(full, spec, jg.SolveOptions(dim=dim), device=dev)
        part = full.leading_objects(n - 1)
        pr = jg.fjofc_embed(part, spec, jg.SolveOptions(dim=dim, init=jg.InitKind.provided,
                                                        init_config=fr.config[:, : n - 1]),
                            device=dev)
        od = delta[:, : n - 1, n - 1]
        res = jg.oos_embed(pr.config, od, 1.0, jg.OosOptions(), seed, device=dev)
        total += float(np.sum(np.linalg.norm(fr.config[:, n - 1] - res.y, axis=1)))
    assert total / 5.0 <= 0.3, total / 5.0
