"""The persistent out-of-sample solve (jofc_oos_solve_kernel) at the
batch shapes its layout plan branches on, against the oracle's oos loop
(proj/src/oos.cpp:180-229 per point): one point per CTA, several point slots per
CTA, more CTAs than SMs (several waves), every d, odd n, zero-distance rows, the
stop rule, and the fallback to the per-update kernels when the plan does not fit."""
import numpy as np
import pytest

import paper_1502_03391_b200 as jg
from conftest import rel_fro
from oracle.oracle import Port

pytestmark = pytest.mark.gpu

X_TOL, S_TOL = 1e-8, 1e-10


@pytest.fixture(scope="module")
def dev():
    d = jg.Device(0)
    d.set_oos_route(1)  # the persistent solve for every shape (AUTO takes it only for full batches)
    yield d
    d.close()


def batch(seed, k, m, n, d, noise=0.05):
    rng = np.random.default_rng(seed)
    x = rng.normal(size=(m, n, d))
    yt = rng.normal(size=(k, m, d))
    od = np.stack([[np.sqrt(((x[l] - yt[q, l]) ** 2).sum(1)) + noise * rng.random(n)
                    for l in range(m)] for q in range(k)])
    y0 = np.stack([jg.oos_start(x, seed + q) for q in range(k)])
    return x, od, y0


def check(dev, x, od, y0, w, eps, its, fixed, sample=None):
    y, tr, it = jg.oos_embed_batch(x, od, w, y0, jg.OosOptions(eps, its), fixed_iterations=fixed,
                                   device=dev)
    idx = np.arange(len(y0)) if sample is None else sample
    yr, trr, itr = Port().oos_batch(x, od[idx], w, y0[idx], eps, its, fixed=fixed)
    for j, q in enumerate(idx):
        assert it[q] == itr[j], (q, it[q], itr[j])
        assert rel_fro(y[q], yr[j]) < X_TOL, q
        t = int(itr[j]) + 1
        assert np.max(np.abs(tr[q, :t] - trr[j, :t]) / np.abs(trr[j, :t])) < S_TOL, q


@pytest.mark.parametrize("k,m,n,d", [
    (1, 2, 777, 3),      # one point, one CTA
    (300, 3, 301, 2),    # 2-3 points per CTA: several slots, odd n
    (5000, 2, 200, 3),   # G = 32 points per CTA: every slot of every warp in use
    (6000, 2, 130, 2),   # more CTAs than SMs: several waves
])
def test_persistent_fixed_count_shapes(dev, k, m, n, d):
    x, od, y0 = batch(k + n, k, m, n, d)
    sample = np.unique(np.linspace(0, k - 1, min(k, 97)).astype(int))
    check(dev, x, od, y0, 0.6, 1e-300, 25, True, sample)


@pytest.mark.parametrize("d", list(range(1, 11)))
def test_persistent_every_dim_with_stop_rule(dev, d):
    x, od, y0 = batch(40 + d, 150, 2, 257, d)
    check(dev, x, od, y0, 0.5, 1e-9, 60, False)


def test_persistent_zero_distance_rows(dev):
    # a point starting exactly on in-sample rows of every modality: dist == 0
    # there (proj/src/oos.cpp:88 ratio 0), the rest of the pass as usual
    x, od, y0 = batch(7, 64, 2, 500, 3)
    y0[5] = x[:, 17, :]
    y0[9] = x[:, 3, :]
    check(dev, x, od, y0, 0.5, 1e-300, 10, True)


def test_persistent_matches_per_update_kernels(dev):
    # the same batch through the per-update fused step kernel
    x, od, y0 = batch(11, 400, 2, 600, 3)
    y, tr, it = jg.oos_embed_batch(x, od, 0.5, y0, jg.OosOptions(1e-300, 30), fixed_iterations=True,
                                   device=dev)
    other = jg.Device(0)
    try:
        other.set_oos_route(2)
        y2, tr2, it2 = jg.oos_embed_batch(x, od, 0.5, y0, jg.OosOptions(1e-300, 30),
                                          fixed_iterations=True, device=other)
    finally:
        other.close()
    assert np.all(it == it2)
    assert rel_fro(y, y2) < 1e-12
    assert np.max(np.abs(tr - tr2) / np.abs(tr2)) < 1e-12


def test_auto_route_matches(dev):
    # AUTO picks the persistent solve for a full batch and the per-update
    # kernels for a small one; both agree with the forced route
    for k in (2000, 40):
        x, od, y0 = batch(13 + k, k, 2, 300, 3)
        y, tr, _ = jg.oos_embed_batch(x, od, 0.5, y0, jg.OosOptions(1e-300, 15),
                                      fixed_iterations=True, device=dev)
        other = jg.Device(0)
        try:
            ya, tra, _ = jg.oos_embed_batch(x, od, 0.5, y0, jg.OosOptions(1e-300, 15),
                                            fixed_iterations=True, device=other)
        finally:
            other.close()
        assert rel_fro(y, ya) < 1e-12
        assert np.max(np.abs(tr - tra) / np.abs(tra)) < 1e-12


def test_route_argument_checked(dev):
    with pytest.raises(ValueError):
        dev.set_oos_route(7)


def test_persistent_falls_back_when_x_chunks_do_not_fit(dev):
    # d = 10 with a large batch per CTA still runs (smaller chunks or the
    # per-update kernels) and matches
    x, od, y0 = batch(3, 3000, 4, 90, 10)
    sample = np.arange(0, 3000, 151)
    check(dev, x, od, y0, 0.3, 1e-300, 12, True, sample)
