"""The C-native NCCL exchange (csrc/capi_nccl.cu) on ONE GPU.

NCCL does not let two ranks of one communicator share a GPU, so on this
one-GPU box the exchange runs as a one-rank communicator: the reduce-scatter,
fidelity all-reduce and all-gather are real NCCL calls on the context stream
(captured in the solve's CUDA graph, or issued per iteration on the stream
route), the epilogue mixes its row chunk (here: every row).  The multi-rank
decomposition itself is checked over gloo in tests/test_layout_shards.py."""
import ctypes as C

import numpy as np
import pytest

import paper_1502_03391_b200 as jg
from paper_1502_03391_b200 import workloads
from paper_1502_03391_b200._capi import check, dptr

pytestmark = pytest.mark.gpu


def solve(dev, wl, prob, its=40):
    opt = jg.SolveOptions(dim=wl.d, eps=1e-300, max_iterations=its, init=jg.InitKind.provided,
                          init_config=wl.x0())
    return jg.fjofc_embed(prob, wl.spec, opt, device=dev)


@pytest.mark.parametrize("direct", [True, False])
@pytest.mark.parametrize("cfg,n", [(5, 1500), (2, 700), (1, 500), (3, 1200)])
def test_one_rank_nccl_matches_unsharded(cfg, n, direct):
    # direct: per-pair fidelity on both sides (same sums, 1e-12); auto: the
    # NCCL route's identity-form fidelity (folded sums all-reduced, decision
    # kernel) against the unsharded per-pair or identity form (1e-10, the
    # north star's stress bound)
    wl = workloads.make(cfg, n=n)
    prob = jg.OmnibusProblem(list(wl.dense_delta()), validate=False)
    ref_dev = jg.Device(0)
    ref_dev.set_fidelity_form(direct=True)
    plain = solve(ref_dev, wl, prob)
    dev = jg.Device(0)
    dev.set_fidelity_form(direct=direct)
    dev.nccl_init(jg.Device.nccl_unique_id(), 0, 1)
    l0 = dev.launches()
    got = solve(dev, wl, prob)
    assert dev.launches() > l0
    assert got.iterations == plain.iterations
    assert np.linalg.norm(got.config - plain.config) <= 1e-12 * np.linalg.norm(plain.config)
    tol = 1e-12 if direct else 1e-10
    assert np.allclose(got.stress_trace, plain.stress_trace, rtol=tol, atol=0)
    dev.close()
    ref_dev.close()


def test_one_rank_nccl_stream_route_and_release():
    # profiling forces per-iteration stream launches (no graph): the NCCL calls
    # are then issued by the C++ loop each iteration
    wl = workloads.make(5, n=1200)
    dev = jg.Device(0)
    dev.upload_features(wl.in_features)
    x0 = wl.x0()
    lib = dev.lib

    def run():
        check(lib.jofc_fjofc_enqueue(dev.h, C.byref(wl.spec.c()), wl.d, dptr(x0), 1e-300, 25))
        x = np.empty_like(x0)
        its, conv = C.c_size_t(), C.c_int()
        check(lib.jofc_fetch_result(dev.h, dptr(x), None, C.byref(its), C.byref(conv)))
        return x, its.value

    ref, _ = run()
    dev.nccl_init(jg.Device.nccl_unique_id(), 0, 1)
    check(lib.jofc_profile(dev.h, 1))
    x, its = run()
    ms, nl = C.c_double(), C.c_uint64()
    check(lib.jofc_profile_read(dev.h, C.byref(ms), C.byref(nl)))
    check(lib.jofc_profile(dev.h, 0))
    assert its == 25 and nl.value == 26
    assert np.linalg.norm(x - ref) <= 1e-12 * np.linalg.norm(ref)
    dev.nccl_release()
    x2, _ = run()
    assert np.linalg.norm(x2 - ref) <= 1e-12 * np.linalg.norm(ref)
    dev.close()


def test_nccl_init_checks():
    dev = jg.Device(0, shard=(1, 2))
    with pytest.raises(jg.InvalidArgument):
        dev.nccl_init(jg.Device.nccl_unique_id(), 0, 2)  # not this context's rank
    with pytest.raises(jg.InvalidArgument):
        dev.nccl_init(b"x" * 10, 1, 2)
    dev.close()
