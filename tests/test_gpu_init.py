"""GPU initialisation against the real reference:
cmds (proj/src/init.cpp:21-42), averaged_procrustes_init (:57-88) and
fjofc_embed with the default InitKind."""
import os

import numpy as np
import pytest

import paper_1502_03391_b200 as jg
from conftest import rel_fro
from oracle.oracle import REF_SO, Port, Spec

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not os.path.exists(REF_SO), reason="oracle/_ref not built")]


@pytest.fixture(scope="module")
def R():
    from oracle.oracle import Reference
    return Reference()


def problem(n, m=2, seed=3, p=4):
    P = Port()
    rng = np.random.default_rng(seed)
    z = rng.normal(size=(n, p))
    return np.stack([P.distance_matrix(z + 0.1 * rng.normal(size=(n, p))) for _ in range(m)])


@pytest.mark.parametrize("n,tol", [(40, 1e-12), (300, 1e-12), (500, 1e-7), (1200, 1e-7)])
def test_cmds_matches_reference(R, n, tol):
    delta = problem(n)
    prob = jg.OmnibusProblem(list(delta), validate=False)
    for d in (1, 2, 3):
        ref = R.cmds(delta, 0, d)
        got = jg.cmds(prob, 0, d)
        assert rel_fro(got, ref) < tol, (n, d, rel_fro(got, ref))


@pytest.mark.parametrize("n,tol", [(60, 1e-12), (400, 1e-7)])
def test_averaged_procrustes_init_matches_reference(R, n, tol):
    delta = problem(n, m=3, seed=9)
    prob = jg.OmnibusProblem(list(delta), validate=False)
    ref = R.averaged_procrustes_init(delta, 2)
    got = jg.averaged_procrustes_init(prob, 2)
    assert rel_fro(got, ref) < tol, rel_fro(got, ref)


def test_default_init_solve_matches_reference(R):
    delta = problem(250, m=2, seed=11)
    prob = jg.OmnibusProblem(list(delta), validate=False)
    opt = jg.SolveOptions(dim=2, eps=1e-300, max_iterations=40)  # default InitKind
    got = jg.fjofc_embed(prob, jg.WeightSpec.uniform(0.5), opt)
    ref = R.fjofc_embed_default_init(delta, Spec.uniform(0.5), 2, 1e-300, 40)
    assert got.iterations == ref.iterations
    assert rel_fro(got.config, ref.x) < 1e-8
    assert max(abs(a - b) / abs(b) for a, b in zip(got.stress_trace, ref.trace)) < 1e-10


@pytest.mark.parametrize("d", [5, 10])
def test_cmds_average_wide_panel(R, d):
    # the modality average (as averaged_procrustes_init builds it) and the
    # widest panels p = d + 4 up to 14
    delta = problem(700, m=3, seed=5, p=12)
    prob = jg.OmnibusProblem(list(delta), validate=False)
    ref = R.cmds(delta, -1, d)
    got = jg.cmds(prob, -1, d)
    assert rel_fro(got, ref) < 1e-7, rel_fro(got, ref)


def test_cmds_low_rank(R):
    # collinear objects: S has rank 1, the trailing eigenpairs are degenerate
    # (null space) and clamp to zero columns
    P = Port()
    rng = np.random.default_rng(21)
    t = rng.normal(size=(400, 1))
    feats = np.hstack([t, 2.0 * t])
    delta = np.stack([P.distance_matrix(feats), P.distance_matrix(1.5 * feats)])
    prob = jg.OmnibusProblem(list(delta), validate=False)
    for modality in (0, -1):
        ref = R.cmds(delta, modality, 3)
        got = jg.cmds(prob, modality, 3)
        assert rel_fro(got, ref) < 1e-7, (modality, rel_fro(got, ref))


@pytest.mark.parametrize("n,m,d,tol", [(60, 3, 2, 1e-12), (150, 2, 3, 1e-12),
                                       (400, 2, 2, 1e-7), (300, 3, 3, 1e-7)])
def test_imputed_omnibus_init_matches_reference(R, n, m, d, tol):
    delta = problem(n, m=m, seed=n + m)
    prob = jg.OmnibusProblem(list(delta), validate=False)
    ref = R.imputed_omnibus_init(delta, d)
    got = jg.imputed_omnibus_init(prob, d)
    assert rel_fro(got, ref) < tol, rel_fro(got, ref)


def test_imputed_dense_cap(R):
    delta = problem(100, m=2, seed=1)
    prob = jg.OmnibusProblem(list(delta), validate=False)
    with pytest.raises(jg.InvalidArgument, match="mn exceeds the dense cap"):
        jg.imputed_omnibus_init(prob, 2, dense_cap=150)
    opt = jg.SolveOptions(dim=2, eps=1e-300, max_iterations=20, init=jg.InitKind.imputed_cmds)
    got = jg.fjofc_embed(prob, jg.WeightSpec.uniform(1.0), opt)
    x0 = R.imputed_omnibus_init(delta, 2)
    ref = R.fjofc_embed(delta, Spec.uniform(1.0), x0, 1e-300, 20)
    assert rel_fro(got.config, ref.x) < 1e-8


@pytest.mark.parametrize("n,k,kind", [(50, 3, "psd"), (400, 3, "indef"), (1500, 5, "psd"),
                                      (700, 6, "indef"), (700, 10, "psd"), (300, 1, "zero")])
def test_symmetric_top_eigenpairs_subspace(R, n, k, kind):
    rng = np.random.default_rng(n + k)
    if kind == "zero":
        s = np.zeros((n, n))
    else:
        a = rng.normal(size=(n, 12))
        s = a @ a.T if kind == "psd" else a @ np.diag(np.linspace(-3, 5, 12)) @ a.T
        s = 0.5 * (s + s.T)
    rv, rvec = R.symmetric_top_eigenpairs_subspace(s, k)
    gv, gvec = jg.symmetric_top_eigenpairs_subspace(s, k)
    scale = max(1.0, float(np.max(np.abs(rv))))
    assert np.max(np.abs(gv - rv)) <= 1e-9 * scale, (gv, rv)
    if kind != "zero":  # top-k inside the 8 (12) nonzero, distinct eigenvalues
        assert rel_fro(gvec, rvec) < 1e-6, rel_fro(gvec, rvec)
    with pytest.raises(jg.InvalidArgument):
        jg.symmetric_top_eigenpairs_subspace(s, n + 1)
