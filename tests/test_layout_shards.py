"""Packed layout and multi-GPU sharding, host side (CPU).

* the stream enumerates every upper-triangle pair exactly once;
* shard ranges partition the stream and balance the estimated cost;
* a world_size-2 gloo run: each rank forms the partial B(X)X products and
  fidelity of ITS blocks only (numpy emulation of the pass kernel's
  arithmetic contract), all-reduces them, applies the W^-1 mix, and must
  reproduce the oracle's guttman_step_fast and raw_stress.
"""
import os

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1502_03391_b200 import layout


@pytest.mark.parametrize("n", [2, 3, 63, 64, 65, 127, 128, 129, 200, 1000])
def test_stream_covers_upper_triangle_once(n):
    seen = np.zeros((n, n), dtype=np.int32)
    for _, B, J in layout.blocks(1, n):
        r0, c0 = B * layout.ROWS, J * layout.COLS
        for i in range(r0, min(r0 + layout.ROWS, n)):
            j0 = max(c0, i + 1)
            j1 = min(c0 + layout.COLS, n)
            if j1 > j0:
                seen[i, j0:j1] += 1
    assert np.array_equal(seen, np.triu(np.ones((n, n), dtype=np.int32), 1))


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_shards_partition_and_balance(world):
    m, n = 2, 20000
    ranges = [layout.shard_range(m, n, r, world) for r in range(world)]
    assert ranges[0][0] == 0 and ranges[-1][1] == m * layout.geometry(n)[2]
    for a, b in zip(ranges, ranges[1:]):
        assert a[1] == b[0]
    # balanced by estimated cost (block_cost), not block count: no shard more
    # than one block's (+ one band entry's) cost above the mean
    nT, nB, _ = layout.geometry(n)
    cost = [layout.block_cost(n, B, J, J == 2 * B)
            for _ in range(m) for B in range(nB) for J in range(2 * B, nT)]
    shares = [sum(cost[lo:hi]) for lo, hi in ranges]
    mean = sum(cost) / world
    assert max(shares) - mean <= 1.0 + layout.MASK_COST + layout.BAND_COST


def partial_products(delta, x, within, m, n, rank, world):
    """Row- and column-side B(X)X partials + weighted fidelity of one shard."""
    P = np.zeros_like(x)
    fid = 0.0
    for l, B, J in layout.blocks(m, n, rank, world):
        r0, c0 = B * layout.ROWS, J * layout.COLS
        rows = np.arange(r0, min(r0 + layout.ROWS, n))
        cols = np.arange(c0, min(c0 + layout.COLS, n))
        if len(rows) == 0 or len(cols) == 0:
            continue
        I, Jj = np.meshgrid(rows, cols, indexing="ij")
        mask = I < Jj
        i, j = I[mask], Jj[mask]
        diff = x[l, i] - x[l, j]
        dist = np.sqrt(np.sum(diff * diff, axis=1))
        dl = delta[l, i, j]
        r = np.where(dist > 0, dl / np.where(dist > 0, dist, 1.0), 0.0)
        contrib = r[:, None] * diff
        np.add.at(P[l], i, contrib)
        np.add.at(P[l], j, -contrib)
        fid += within[l] * np.sum((dl - dist) ** 2)
    return P, fid


def _worker(rank, world, port, payload, out):
    import torch
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    delta, x, within, coef, cross = payload
    m, n, d = x.shape
    P, fid = partial_products(delta, x, within, m, n, rank, world)
    buf = torch.from_numpy(np.concatenate([P.ravel(), [fid]]))
    dist.all_reduce(buf)
    red = buf.numpy()
    P, fid = red[:-1].reshape(m, n, d), red[-1]
    xn = np.einsum("jl,lic->jic", coef, P)
    com = sum(cross[a, b] * np.sum((x[a] - x[b]) ** 2)
              for a in range(m) for b in range(a + 1, m))
    out[rank] = (xn, fid + com)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_step_gloo_matches_oracle(world):
    from oracle.oracle import Port, Spec
    P = Port()
    rng = np.random.default_rng(5)
    m, n, d = 2, 300, 3
    delta = np.stack([P.distance_matrix(rng.normal(size=(n, 3))) for _ in range(m)])
    x = rng.normal(size=(m, n, d))
    spec = Spec.uniform(0.5)
    within, cross = P.weights_expand(spec, m)
    winv = P.script_w_inverse(spec, m, n)
    coef = winv * within[None, :]
    mgr = mp.Manager()
    out = mgr.dict()
    port = 29500 + os.getpid() % 1000
    mp.spawn(_worker, args=(world, port, (delta, x, within, coef, cross), out), nprocs=world,
             join=True)
    ref_step = P.guttman_step_fast(delta, spec, x)
    ref_stress = P.raw_stress(delta, spec, x)
    for r in range(world):
        xn, sigma = out[r]
        assert np.linalg.norm(xn - ref_step) / np.linalg.norm(ref_step) < 1e-12
        assert abs(sigma - ref_stress) / ref_stress < 1e-12
    # both ranks hold identical results (the all-reduce is the only exchange)
    assert np.array_equal(out[0][0], out[1][0])


def _peer_worker(rank, world, port, payload, out):
    # the peer exchange's decomposition (csrc/jofc_peer.cuh) restated over
    # gloo: slab handles all-gathered; each rank sums ITS rows of every rank's
    # partial products in rank order, mixes them and writes the rows to every
    # rank; sigma = rank-order sum of the fidelity partials + rank-order sum of
    # the per-rank commensurability
    import torch
    from paper_1502_03391_b200.dist import exchange_handles
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    handles = exchange_handles(bytes([rank + 1]) * 64)
    assert handles == [bytes([q + 1]) * 64 for q in range(world)]
    delta, x, within, coef, cross = payload
    m, n, d = x.shape
    P, fid = partial_products(delta, x, within, m, n, rank, world)
    slabs = [torch.zeros(P.size + 1, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(slabs, torch.from_numpy(np.concatenate([P.ravel(), [fid]])))
    lo, hi = n * rank // world, n * (rank + 1) // world
    S = np.zeros((m, hi - lo, d))
    for q in range(world):
        S += slabs[q].numpy()[:-1].reshape(m, n, d)[:, lo:hi]
    rows = np.einsum("jl,lic->jic", coef, S)
    com = sum(cross[a, b] * np.sum((x[a, lo:hi] - x[b, lo:hi]) ** 2)
              for a in range(m) for b in range(a + 1, m))
    gathered = [None] * world
    dist.all_gather_object(gathered, (lo, hi, rows, com))
    xn = np.zeros_like(x)
    for q_lo, q_hi, q_rows, _ in gathered:
        xn[:, q_lo:q_hi] = q_rows
    sigma = 0.0
    for q in range(world):
        sigma += float(slabs[q][-1])
    comsum = 0.0
    for *_, q_com in gathered:
        comsum += q_com
    out[rank] = (xn, sigma + comsum)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_peer_decomposition_gloo_matches_oracle(world):
    from oracle.oracle import Port, Spec
    P = Port()
    rng = np.random.default_rng(6)
    m, n, d = 3, 257, 2
    delta = np.stack([P.distance_matrix(rng.normal(size=(n, 3))) for _ in range(m)])
    x = rng.normal(size=(m, n, d))
    spec = Spec.uniform(0.7)
    within, cross = P.weights_expand(spec, m)
    winv = P.script_w_inverse(spec, m, n)
    coef = winv * within[None, :]
    mgr = mp.Manager()
    out = mgr.dict()
    port = 30500 + os.getpid() % 1000
    mp.spawn(_peer_worker, args=(world, port, (delta, x, within, coef, cross), out),
             nprocs=world, join=True)
    ref_step = P.guttman_step_fast(delta, spec, x)
    ref_stress = P.raw_stress(delta, spec, x)
    for r in range(world):
        xn, sigma = out[r]
        assert np.linalg.norm(xn - ref_step) / np.linalg.norm(ref_step) < 1e-12
        assert abs(sigma - ref_stress) / ref_stress < 1e-12
    assert np.array_equal(out[0][0], out[1][0]) and out[0][1] == out[1][1]


def _nccl_worker(rank, world, port, payload, out):
    # the C-native NCCL exchange (csrc/capi_nccl.cu) restated over gloo: P in
    # the device layout (m x n_pad x d), an in-place reduce-scatter of each
    # modality's row chunks (gloo has no reduce_scatter: all-reduce + own
    # chunk, the same values), a fidelity all-reduce, the W^-1 mix of the OWN
    # chunk's objects only, commensurability of the replicated X_t over all
    # objects (every rank, same order), an all-gather of X_{t+1} row chunks;
    # and the identity-form sigma from the all-reduced own-row sums
    import torch
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    delta, x, within, coef, cross = payload
    m, n, d = x.shape
    n_pad = layout.ROWS * layout.geometry(n)[1]
    assert n_pad % world == 0
    chunk = n_pad // world
    P, fid = partial_products(delta, x, within, m, n, rank, world)
    Pd = np.zeros((m, n_pad, d))
    Pd[:, :n] = P
    own = slice(rank * chunk, (rank + 1) * chunk)
    for l in range(m):  # reduce-scatter of modality l's row chunks
        t = torch.from_numpy(Pd[l].copy())
        dist.all_reduce(t)
        Pd[l, own] = t.numpy()[own]
    f = torch.tensor([fid], dtype=torch.float64)
    dist.all_reduce(f)
    lo, hi = min(n, rank * chunk), min(n, (rank + 1) * chunk)
    xn = np.zeros((m, n_pad, d))
    xn[:, lo:hi] = np.einsum("jl,lic->jic", coef, Pd[:, lo:hi])
    com = sum(cross[a, b] * np.sum((x[a] - x[b]) ** 2) for a in range(m) for b in range(a + 1, m))
    # identity-form fidelity (csrc/jofc_kernels.cuh rho_fold / rho_decide):
    # each rank folds, over ITS rows only, the commensurability and per
    # modality R = x_i . P_i (reduced P rows), Q = |x_i - x_0|^2, its shard's
    # A = sum of its stored delta^2, C = x_i - x_0; the vector rides in the
    # all-gather group as one all-reduce
    A = shard_sumsq(delta, m, n, rank, world)
    vec = [sum(cross[a, b] * np.sum((x[a, lo:hi] - x[b, lo:hi]) ** 2)
               for a in range(m) for b in range(a + 1, m))]
    for l in range(m):
        dx = x[l, lo:hi] - x[l, 0]
        vec += [float(np.sum(x[l, lo:hi] * Pd[l, lo:hi])), float(np.sum(dx * dx)), A[l]]
        vec += list(dx.sum(0))
    for l in range(m):  # all-gather of X_{t+1} row chunks
        parts = [torch.zeros(chunk, d, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, torch.from_numpy(xn[l, own].copy()))
        xn[l] = torch.cat(parts).numpy()
    v = torch.tensor(vec, dtype=torch.float64)
    dist.all_reduce(v)
    v = v.numpy()
    sig_rho = v[0]
    for l in range(m):
        R, Q, Al = v[1 + l * (d + 3): 4 + l * (d + 3)]
        C = v[4 + l * (d + 3): 1 + (l + 1) * (d + 3)]
        sig_rho += within[l] * (Al + (n * Q - C @ C) - 2 * R)
    out[rank] = (xn[:, :n], float(f[0]) + com, sig_rho)
    dist.destroy_process_group()


def shard_sumsq(delta, m, n, rank, world):
    """A_l over one shard's blocks (jofc_modality_sumsq_kernel)."""
    A = np.zeros(m)
    for l, B, J in layout.blocks(m, n, rank, world):
        r0, c0 = B * layout.ROWS, J * layout.COLS
        for i in range(r0, min(r0 + layout.ROWS, n)):
            j0, j1 = max(c0, i + 1), min(c0 + layout.COLS, n)
            if j1 > j0:
                A[l] += np.sum(delta[l, i, j0:j1] ** 2)
    return A


@pytest.mark.parametrize("world", [2, 4])
def test_nccl_native_decomposition_gloo_matches_oracle(world):
    from oracle.oracle import Port, Spec
    P = Port()
    rng = np.random.default_rng(7)
    m, n, d = 3, 300, 3
    delta = np.stack([P.distance_matrix(rng.normal(size=(n, 3))) for _ in range(m)])
    x = rng.normal(size=(m, n, d))
    spec = Spec.uniform(0.6)
    within, cross = P.weights_expand(spec, m)
    coef = P.script_w_inverse(spec, m, n) * within[None, :]
    mgr = mp.Manager()
    out = mgr.dict()
    port = 31500 + os.getpid() % 1000 + world
    mp.spawn(_nccl_worker, args=(world, port, (delta, x, within, coef, cross), out),
             nprocs=world, join=True)
    ref_step = P.guttman_step_fast(delta, spec, x)
    ref_stress = P.raw_stress(delta, spec, x)
    for r in range(world):
        xn, sigma, sigma_rho = out[r]
        assert np.linalg.norm(xn - ref_step) / np.linalg.norm(ref_step) < 1e-12
        assert abs(sigma - ref_stress) / ref_stress < 1e-12
        assert abs(sigma_rho - ref_stress) / ref_stress < 1e-12
    for r in range(1, world):  # replicated X and stop state on every rank
        assert np.array_equal(out[r][0], out[0][0]) and out[r][1:] == out[0][1:]
