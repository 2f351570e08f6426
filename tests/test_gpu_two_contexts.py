"""Two contexts on one GPU, double-buffered the way bench.py's e2e drives them
(run_e2e_pipelined): the dense host Delta of one problem is uploaded
(jofc_set_problem) on context B while context A's enqueued solve is still
running, B's solve is enqueued behind it, then A's result is fetched.  Each
context owns its packed Delta, iterates, control block and streams, so every
result must match the same solve run alone on a fresh context, and the
reference oracle."""
import ctypes as C

import numpy as np
import pytest

import paper_1502_03391_b200 as jg
from oracle.oracle import Port, Spec
from paper_1502_03391_b200 import workloads
from paper_1502_03391_b200._capi import _dp, check, dptr

pytestmark = pytest.mark.gpu


def upload(dev, delta):
    m, n = delta.shape[0], delta.shape[1]
    ptrs = (_dp * m)(*[dptr(delta[l]) for l in range(m)])
    check(dev.lib.jofc_set_problem(dev.h, m, n, ptrs, 0))


def enqueue(dev, spec, d, x0, max_it):
    check(dev.lib.jofc_fjofc_enqueue(dev.h, C.byref(spec.c()), d, dptr(x0), 1e-300, max_it))


def fetch(dev, shape, max_it):
    x = np.empty(shape)
    trace = np.empty(max_it + 1)
    its, conv = C.c_size_t(), C.c_int()
    check(dev.lib.jofc_fetch_result(dev.h, dptr(x), dptr(trace), C.byref(its), C.byref(conv)))
    return x, trace[: its.value + 1].copy(), its.value


@pytest.mark.parametrize("cfg,n", [(5, 3000), (2, 700)])  # stream/graph route, single launch
def test_upload_under_other_contexts_solve(cfg, n):
    T = 30
    wls = [workloads.make(cfg, n=n, seed=s) for s in (11, 12, 13, 14)]
    deltas = [np.ascontiguousarray(w.dense_delta()) for w in wls]
    x0s = [w.x0() for w in wls]
    spec = wls[0].spec
    d = wls[0].d
    # alone: one fresh context per problem
    alone = []
    for delta, x0 in zip(deltas, x0s):
        dev = jg.Device(0)
        upload(dev, delta)
        enqueue(dev, spec, d, x0, T)
        alone.append(fetch(dev, x0.shape, T))
        dev.close()
    # double-buffered over two contexts
    devs = [jg.Device(0), jg.Device(0)]
    got = [None] * len(deltas)
    upload(devs[0], deltas[0])
    enqueue(devs[0], spec, d, x0s[0], T)
    for k in range(1, len(deltas)):
        upload(devs[k & 1], deltas[k])        # while solve k-1 runs on the other context
        enqueue(devs[k & 1], spec, d, x0s[k], T)
        got[k - 1] = fetch(devs[(k - 1) & 1], x0s[k - 1].shape, T)
    got[-1] = fetch(devs[(len(deltas) - 1) & 1], x0s[-1].shape, T)
    for dv in devs:
        dv.close()
    ospec = Spec.general_(spec.general) if wls[0].general_weights else Spec.uniform(wls[0].w)
    for k, ((x, tr, its), (xa, tra, itsa)) in enumerate(zip(got, alone)):
        assert its == itsa == T
        # column-side products use RED atomics: equal to rounding, not bitwise
        assert np.linalg.norm(x - xa) <= 1e-12 * np.linalg.norm(xa), k
        assert np.all(np.abs(tr - tra) <= 1e-12 * np.abs(tra)), k
    # and the first problem against the CPU oracle
    ref = Port().fjofc_embed(deltas[0], ospec, x0s[0], 1e-300, T)
    assert np.linalg.norm(got[0][0] - ref.x) <= 1e-8 * np.linalg.norm(ref.x)
    assert np.all(np.abs(got[0][1] - ref.trace) <= 1e-10 * np.abs(ref.trace))
