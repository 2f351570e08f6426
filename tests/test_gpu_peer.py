"""Peer-memory exchange (csrc/jofc_peer.cuh) on ONE GPU.

W contexts own disjoint shards of the same problem and exchange products and
configuration rows through each other's slabs (device pointers: contexts of
one process).  jofc_peer_lockstep_solve launches stage by stage with stream
events between the ranks' stages, so every flag a kernel polls was raised
before it starts: the kernels and the protocol (parity of the P regions,
flags, epochs, rank-order sums) run as on W GPUs, but no kernel waits for
another one that is still running.  Every rank must reproduce the unsharded
solve and hold bitwise-identical iterates."""
import numpy as np
import pytest

import paper_1502_03391_b200 as jg
from paper_1502_03391_b200 import workloads

pytestmark = pytest.mark.gpu


def group(prob, world):
    devs = [jg.Device(0, shard=(r, world)) for r in range(world)]
    for dv in devs:
        dv.upload(prob)
    slabs = [dv.peer_export()[1] for dv in devs]
    for r, dv in enumerate(devs):
        dv.peer_attach_pointers(r, world, slabs)
    return devs


def check_against_single(out, single):
    x_ref = single.config
    for x, trace, its, _ in out:
        assert its == single.iterations
        k = its
        assert np.linalg.norm(x - x_ref) / np.linalg.norm(x_ref) < 1e-12
        ref = np.asarray(single.stress_trace[: k + 1])
        assert np.all(np.abs(trace[: k + 1] - ref) <= 1e-12 * np.abs(ref))
    for x, trace, its, _ in out[1:]:  # rank-order sums: identical on every rank
        assert np.array_equal(x, out[0][0])
        assert np.array_equal(trace, out[0][1]) and its == out[0][2]


@pytest.mark.parametrize("world", [2, 3, 4])
def test_peer_lockstep_matches_single(world):
    wl = workloads.make(5, n=700)
    x0 = wl.x0()
    prob = jg.OmnibusProblem(list(wl.dense_delta()), validate=False)
    opt = jg.SolveOptions(dim=wl.d, eps=1e-300, max_iterations=15, init=jg.InitKind.provided,
                          init_config=x0)
    single = jg.fjofc_embed(prob, wl.spec, opt, device=jg.Device(0))
    devs = group(prob, world)
    out = jg.peer_lockstep_solve(devs, wl.spec, x0, 1e-300, 15)
    check_against_single(out, single)


def test_peer_lockstep_many_modalities_and_ragged_rows():
    # m = 4 (mix over four products per object), n not a multiple of the
    # world or of 64, general weights
    rng = np.random.default_rng(11)
    m, n, d, world = 4, 333, 3, 3
    feats = [rng.normal(size=(n, 3)) for _ in range(m)]
    delta = [np.sqrt(((f[:, None] - f[None]) ** 2).sum(-1)) for f in feats]
    prob = jg.OmnibusProblem(delta, validate=False)
    g = np.array([[1.0 + 0.2 * i if i == j else 0.3 + 0.1 * abs(i - j) for j in range(m)]
                  for i in range(m)])
    spec = jg.WeightSpec.general(g)
    x0 = rng.normal(size=(m, n, d))
    opt = jg.SolveOptions(dim=d, eps=1e-300, max_iterations=9, init=jg.InitKind.provided,
                          init_config=x0)
    single = jg.fjofc_embed(prob, spec, opt, device=jg.Device(0))
    out = jg.peer_lockstep_solve(group(prob, world), spec, x0, 1e-300, 9)
    check_against_single(out, single)


def test_peer_successive_solves():
    # consecutive solves on the same slabs: the P region parity carries over
    # from the previous solve's last iteration (odd and even counts, an eps
    # stop, a dimension change), the flags over the epochs
    wl = workloads.make(1, n=300)
    prob = jg.OmnibusProblem(list(wl.dense_delta()), validate=False)
    devs = group(prob, 2)
    rng = np.random.default_rng(3)
    m, n = wl.m, wl.n
    for d, eps, T in [(2, 1e-300, 7), (3, 1e-300, 4), (2, 1e-4, 60), (1, 1e-300, 5),
                      (2, 1e-300, 0), (3, 1e-300, 6)]:
        x0 = rng.normal(size=(m, n, d))
        opt = jg.SolveOptions(dim=d, eps=eps, max_iterations=T, init=jg.InitKind.provided,
                              init_config=x0)
        single = jg.fjofc_embed(prob, wl.spec, opt, device=jg.Device(0))
        out = jg.peer_lockstep_solve(devs, wl.spec, x0, eps, T)
        check_against_single(out, single)
        if eps > 1e-200:
            assert out[0][2] < T  # the stop rule fired


def test_peer_export_and_attach_checks():
    wl = workloads.make(1, n=200)
    prob = jg.OmnibusProblem(list(wl.dense_delta()), validate=False)
    dv = jg.Device(0, shard=(0, 2))
    dv.upload(prob)
    with pytest.raises(jg.InvalidArgument):
        dv.peer_attach_pointers(0, 2, [0, 0])  # nothing exported yet
    handle, slab = dv.peer_export()
    assert len(handle) == 64 and slab
    with pytest.raises(jg.InvalidArgument):
        dv.peer_attach_pointers(1, 2, [slab, slab])  # not this context's rank
    with pytest.raises(jg.InvalidArgument):
        dv.peer_attach_pointers(0, 2, [0, slab])  # slab 0 is not this context's
    with pytest.raises(jg.InvalidArgument):
        dv.peer_attach_pointers(0, 1, [slab])  # one rank has nothing to exchange
    # a detached context is back on the all-reduce hook (none set: loud error)
    other = jg.Device(0, shard=(1, 2))
    other.upload(prob)
    dv.peer_attach_pointers(0, 2, [slab, other.peer_export()[1]])
    dv.peer_detach()
    opt = jg.SolveOptions(dim=wl.d, eps=1e-300, max_iterations=2, init=jg.InitKind.provided,
                          init_config=wl.x0())
    with pytest.raises(jg.CommError):
        jg.fjofc_embed(prob, wl.spec, opt, device=dv)


def test_peer_missing_rank_fails_loudly():
    # rank 1 never runs: rank 0's exchange kernel gives up after its 20 s
    # timeout and the solve raises instead of hanging (no kernel waits on a
    # running kernel: the other rank is simply absent)
    wl = workloads.make(1, n=200)
    prob = jg.OmnibusProblem(list(wl.dense_delta()), validate=False)
    devs = group(prob, 2)
    opt = jg.SolveOptions(dim=wl.d, eps=1e-300, max_iterations=2, init=jg.InitKind.provided,
                          init_config=wl.x0())
    with pytest.raises(jg.CommError, match="did not arrive"):
        jg.fjofc_embed(prob, wl.spec, opt, device=devs[0])


def _ipc_worker(rank, world, port, out):
    # the production attach path: slabs exported as CUDA IPC handles, handles
    # all-gathered over torch.distributed (gloo), the other rank's slab opened;
    # each rank then writes a marker into its own slab and reads the other's
    # through its mapping (plain copies: no kernel waits on another)
    import os

    import torch
    import torch.distributed as dist

    from paper_1502_03391_b200.dist import attach_peers, cuda_view
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    wl = workloads.make(1, n=200)
    dev = jg.Device(0, shard=(rank, world))
    dev.upload(jg.OmnibusProblem(list(wl.dense_delta()), validate=False))
    handles = attach_peers(dev)
    assert len(handles) == world and all(len(h) == 64 for h in handles)
    own = dev.lib.jofc_peer_address(dev.h, rank)
    other = dev.lib.jofc_peer_address(dev.h, 1 - rank)
    assert own and other and own != other
    cuda_view(own, 8, "cuda:0").copy_(
        torch.full((8,), 1.5 * (rank + 1), dtype=torch.float64, device="cuda:0"))
    torch.cuda.synchronize()
    dist.barrier()
    out[rank] = cuda_view(other, 8, "cuda:0").cpu().numpy().tolist()
    dist.barrier()
    dev.close()
    dist.destroy_process_group()


def test_peer_ipc_attach_two_processes():
    import os
    import socket

    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_ipc_worker, args=(2, port, out), nprocs=2, join=True)
    assert out[0] == [3.0] * 8 and out[1] == [1.5] * 8, dict(out)
