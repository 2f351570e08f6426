"""Identity-form fidelity (csrc/jofc_kernels.cuh, rho_decide) against the
reference library and against the per-pair form, on the one-GPU route it
applies to (separate epilogue kernel: n > 1024, stream launches or the CUDA
graph), including the switch to the per-pair sum on close fits.

Tolerances are the north star's (BASELINE.json): X within 1e-8 relative
Frobenius, every stress-trace entry within 1e-10 relative, same iterations.
"""
import numpy as np
import pytest

import paper_1502_03391_b200 as jg
from conftest import rel, rel_fro
from oracle.oracle import Port, Spec, best_available
from paper_1502_03391_b200 import workloads

pytestmark = pytest.mark.gpu

X_TOL = 1e-8
S_TOL = 1e-10


@pytest.fixture
def dev():
    d = jg.Device(0)
    d.profile(True)  # per-iteration stream launches: the identity-form route at small n
    yield d
    d.close()


def _oracle_spec(wl):
    return Spec.general_(wl.spec.general) if wl.general_weights else Spec.uniform(wl.w)


def _solve(dev, delta, spec, x0, iters, eps=1e-300):
    opt = jg.SolveOptions(dim=x0.shape[2], eps=eps, max_iterations=iters,
                          init=jg.InitKind.provided, init_config=x0)
    return jg.fjofc_embed(jg.OmnibusProblem(list(delta), validate=False), spec, opt, device=dev)


def _check(r, ref):
    k = min(len(r.stress_trace), len(ref.trace))
    worst = max(rel(a, b) for a, b in zip(r.stress_trace[:k], ref.trace[:k]))
    assert worst < S_TOL, worst
    assert r.iterations == ref.iterations, (r.iterations, ref.iterations)
    assert rel_fro(r.config, ref.x) < X_TOL
    return worst


@pytest.mark.parametrize("cfg,n,iters", [(3, 2500, 25), (4, 1500, 25), (2, 1200, 40)])
def test_identity_form_against_reference(dev, cfg, n, iters):
    wl = workloads.make(cfg, n=n)
    delta, x0 = wl.dense_delta(), wl.x0()
    ref = best_available().fjofc_embed(delta, _oracle_spec(wl), x0, 1e-300, iters, parallel=True)
    r = _solve(dev, delta, wl.spec, x0, iters)
    _check(r, ref)
    # the per-pair form on the same device agrees with it to the same bound
    dev.set_fidelity_form(direct=True)
    rd = _solve(dev, delta, wl.spec, x0, iters)
    dev.set_fidelity_form(direct=False)
    assert max(rel(a, b) for a, b in zip(r.stress_trace, rd.stress_trace)) < S_TOL
    assert rel_fro(r.config, rd.config) < 1e-11
    # (and the identity form was in use: t >= 1 entries differ in their last bits)
    assert any(a != b for a, b in zip(r.stress_trace[1:], rd.stress_trace[1:]))


def _near_realizable(n, noise, seed):
    rng = np.random.default_rng(seed)
    z = rng.normal(size=(n, 2))
    P = Port()
    delta = np.stack([P.distance_matrix(z + noise * rng.normal(size=(n, 2))) for _ in range(2)])
    return z, delta


def test_close_fit_switches_to_direct_mid_solve(dev):
    # sigma falls from O(1) of sum delta^2 to ~1e-9 of it: the identity form's
    # cancellation would exceed 1e-10 without the switch
    n = 1100
    z, delta = _near_realizable(n, 1e-5, 61)
    x0 = np.stack([z, z]) + np.random.default_rng(62).normal(size=(2, n, 2))
    spec = jg.WeightSpec.uniform(0.5)
    ref = best_available().fjofc_embed(delta, Spec.uniform(0.5), x0, 1e-300, 60, parallel=True)
    r = _solve(dev, delta, spec, x0, 60)
    assert ref.trace[-1] < 1e-6 * ref.trace[0]  # the fit did get close
    _check(r, ref)


def test_close_fit_from_the_start(dev):
    # warm start near the generating configuration: iteration 0 (always per
    # pair) already sees F / (A + S + 2R) ~ 1e-7 < 1e-5, so no iteration uses
    # the identity form (whose error here would be ~4e-9 relative)
    n = 1100
    z, delta = _near_realizable(n, 1e-3, 63)
    x0 = np.stack([z, z]) + 1e-4 * np.random.default_rng(64).normal(size=(2, n, 2))
    spec = jg.WeightSpec.uniform(0.5)
    ref = best_available().fjofc_embed(delta, Spec.uniform(0.5), x0, 1e-300, 10, parallel=True)
    r = _solve(dev, delta, spec, x0, 10)
    _check(r, ref)


def test_stop_rule_iterations_match(dev):
    # the eps rule decides on sigma differences: same stopping iteration as
    # the reference with the identity form in use
    wl = workloads.make(3, n=2000)
    delta, x0 = wl.dense_delta(), wl.x0()
    ref = best_available().fjofc_embed(delta, _oracle_spec(wl), x0, 1e-4, 200, parallel=True)
    assert ref.iterations < 200
    r = _solve(dev, delta, wl.spec, x0, 200, eps=1e-4)
    _check(r, ref)
    assert r.terminated == jg.Termination.converged
