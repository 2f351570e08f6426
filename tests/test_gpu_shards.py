"""Sharded (multi-GPU) data path on ONE GPU: W contexts own disjoint block
ranges of the same problem; partial products are exchanged through the C ABI's
all-reduce hook (ThreadGroup: host-side reduction, no device-side waits) and
every rank must reproduce the unsharded solve."""
import threading

import numpy as np
import pytest

import paper_1502_03391_b200 as jg
from paper_1502_03391_b200 import workloads
from paper_1502_03391_b200.dist import ThreadGroup

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_solve_matches_single(world):
    wl = workloads.make(5, n=700)
    x0 = wl.x0()
    prob = jg.OmnibusProblem(list(wl.dense_delta()), validate=False)
    opt = jg.SolveOptions(dim=wl.d, eps=1e-300, max_iterations=15, init=jg.InitKind.provided,
                          init_config=x0)
    single = jg.fjofc_embed(prob, wl.spec, opt, device=jg.Device(0))

    group = ThreadGroup(world)
    results = [None] * world
    errors = []

    def run(rank):
        try:
            dev = jg.Device(0, shard=(rank, world))
            dev.set_allreduce(group.hook_for(rank, "cuda:0"))
            results[rank] = jg.fjofc_embed(prob, wl.spec, opt, device=dev)
        except Exception as e:  # noqa: BLE001
            errors.append(e)
            group.bar.abort()

    threads = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    for r in range(world):
        res = results[r]
        assert res.iterations == single.iterations
        assert np.linalg.norm(res.config - single.config) / np.linalg.norm(single.config) < 1e-12
        for a, b in zip(res.stress_trace, single.stress_trace):
            assert abs(a - b) <= 1e-12 * abs(b)
    # every rank walked identical iterates (all-reduce output is shared)
    for r in range(1, world):
        assert np.array_equal(results[r].config, results[0].config)


def test_sharded_context_without_hook_fails_loudly():
    wl = workloads.make(1, n=200)
    dev = jg.Device(0, shard=(0, 2))
    prob = jg.OmnibusProblem(list(wl.dense_delta()), validate=False)
    opt = jg.SolveOptions(dim=wl.d, eps=1e-300, max_iterations=3, init=jg.InitKind.provided,
                          init_config=wl.x0())
    with pytest.raises(jg.CommError):
        jg.fjofc_embed(prob, wl.spec, opt, device=dev)
