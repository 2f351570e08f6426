"""Back-to-back asynchronous solves on one context (jofc_fjofc_enqueue): each
solve runs with its OWN control block (eps, max_iterations), even when a later
enqueue with different parameters follows before the first one executes --
the control block is written by a kernel whose parameter carries the values,
not copied from a reused host buffer.  The device counts the iterations each
solve executed (jofc_stress_evaluations)."""
import ctypes as C

import numpy as np
import pytest

import paper_1502_03391_b200 as jg
from paper_1502_03391_b200 import workloads
from paper_1502_03391_b200._capi import check, dptr

pytestmark = pytest.mark.gpu


def enqueue(dev, spec, d, x0, eps, max_it):
    check(dev.lib.jofc_fjofc_enqueue(dev.h, C.byref(spec.c()), d, dptr(x0), eps, max_it))


def fetch(dev, shape):
    x = np.empty(shape)
    its, conv = C.c_size_t(), C.c_int()
    trace = np.empty(1000)
    check(dev.lib.jofc_fetch_result(dev.h, dptr(x), dptr(trace), C.byref(its), C.byref(conv)))
    return x, trace[: its.value + 1].copy(), its.value, conv.value


def solve_alone(dev, spec, d, x0, eps, max_it):
    enqueue(dev, spec, d, x0, eps, max_it)
    return fetch(dev, x0.shape)


@pytest.mark.parametrize("n", [300, 3000])  # persistent single launch / graph + stream route
def test_back_to_back_solves_keep_their_parameters(n):
    wl = workloads.make(5, n=n)
    dev = jg.Device(0)
    dev.upload_features(wl.in_features)
    rng = np.random.default_rng(1)
    xa = rng.normal(size=(wl.m, wl.n, wl.d))
    xb = rng.normal(size=(wl.m, wl.n, wl.d))
    # B: an eps that stops it part way (from its own fixed-count trace)
    full = solve_alone(dev, wl.spec, wl.d, xb, 1e-300, 60)[1]
    mn = wl.m * wl.n
    dec = (full[:-1] - full[1:]) / (mn * (mn - 1) / 2)
    eps = float(dec[20]) * 1.0001
    b_alone = solve_alone(dev, wl.spec, wl.d, xb, eps, 60)
    assert 0 < b_alone[2] < 60 and b_alone[3] == 1
    a_alone = solve_alone(dev, wl.spec, wl.d, xa, 1e-300, 37)
    assert a_alone[2] == 37
    # A (37 fixed iterations) immediately followed by B (eps stop): A must not
    # pick up B's eps / max_it, nor a half-written control block
    e0 = dev.stress_evaluations()
    for _ in range(3):
        enqueue(dev, wl.spec, wl.d, xa, 1e-300, 37)
        enqueue(dev, wl.spec, wl.d, xb, eps, 60)
    x, trace, its, conv = fetch(dev, xb.shape)
    evals = dev.stress_evaluations() - e0
    assert evals == 3 * ((37 + 1) + (b_alone[2] + 1))
    assert its == b_alone[2] and conv == 1
    # (column-side products are added with RED atomics: bitwise equality
    # between two runs is not expected, agreement to rounding is)
    assert np.linalg.norm(x - b_alone[0]) <= 1e-12 * np.linalg.norm(b_alone[0])
    assert np.all(np.abs(trace - b_alone[1]) <= 1e-12 * np.abs(b_alone[1]))
    dev.close()


def test_step_seconds_keeps_single_launch_route():
    wl = workloads.make(1, n=400)
    dev = jg.Device(0)
    prob = jg.OmnibusProblem(list(wl.dense_delta()), validate=False)
    opt = jg.SolveOptions(dim=wl.d, eps=1e-300, max_iterations=20, init=jg.InitKind.provided,
                          init_config=wl.x0())
    l0 = dev.launches()
    r = jg.fjofc_embed(prob, wl.spec, opt, device=dev)
    used = dev.launches() - l0
    assert r.iterations == 20 and len(r.step_seconds) == 20
    assert all(s > 0 for s in r.step_seconds)
    # upload + control block + ONE cooperative solve launch (no per-iteration launches)
    assert used < 20, used
    dev.close()
