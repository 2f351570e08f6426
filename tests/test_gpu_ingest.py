"""Streaming Delta ingest: jofc_load_problem_files
against the real reference's load_dissimilarities (proj/src/io.cpp:152-215)
and .jofc container (proj/src/io.cpp:84-125, 217-229).

Valid inputs: the device-loaded problem must be bit-identical to uploading the
reference-loaded dense matrices: raw_stress (deterministic reduction) compared
with ==, one Guttman transform to 1e-13 (its column sums use atomics, so the
transform itself is reproducible only to rounding).  Invalid inputs: the same
error message."""
import os
import struct
import threading

import numpy as np
import pytest

import paper_1502_03391_b200 as jg
from paper_1502_03391_b200 import workloads
from paper_1502_03391_b200.dist import ThreadGroup
from oracle.oracle import REF_SO, Port

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not os.path.exists(REF_SO), reason="oracle/_ref not built")]


@pytest.fixture(scope="module")
def R():
    from oracle.oracle import Reference
    return Reference()


@pytest.fixture(scope="module")
def dev():
    return jg.Device(0)


def deltas(n, m=2, seed=0, p=3):
    P = Port()
    rng = np.random.default_rng(seed)
    z = rng.normal(size=(n, p))
    return np.stack([P.distance_matrix(z + 0.2 * rng.normal(size=(n, p))) for _ in range(m)])


def write_csv(path, a, fmt="%.17g", sep=",", blank_every=0):
    with open(path, "w") as f:
        for i, row in enumerate(a):
            if blank_every and i % blank_every == 0:
                f.write("  \n")
            f.write(sep.join(fmt % v for v in row) + "\n")


def perturb(a, seed):
    """Asymmetry well inside 1e-9 relative, plus a nonzero diagonal entry."""
    rng = np.random.default_rng(seed)
    b = a.copy()
    n = len(b)
    idx = rng.integers(0, n, size=(3 * n, 2))
    for i, j in idx:
        if i != j:
            b[i, j] = b[i, j] * (1.0 + 3e-10 * rng.uniform(-1, 1))
    b[n // 3, n // 3] = 0.25
    return b


def same_problem(dev_loaded, dense, seed=5, d=3):
    """Bit-identical device problems: loaded from files vs uploaded dense."""
    m, n, _ = dense.shape
    other = jg.Device(0)
    ref_prob = jg.OmnibusProblem(list(dense), validate=False)
    x = np.random.default_rng(seed).normal(size=(m, n, d))
    for spec in (jg.WeightSpec.uniform(0.5), jg.WeightSpec.product([1.0 + 0.5 * i for i in range(m)], 2.0)):
        s1 = jg.raw_stress(x, dev_loaded, spec, device=dev_loaded.device)
        s2 = jg.raw_stress(x, ref_prob, spec, device=other)
        assert s1 == s2, (s1, s2)
        x1 = jg.guttman_step_fast(x, dev_loaded, spec, device=dev_loaded.device)
        x2 = jg.guttman_step_fast(x, ref_prob, spec, device=other)
        np.testing.assert_allclose(x1, x2, rtol=1e-13, atol=1e-13 * np.abs(x2).max())
    other.close()


@pytest.mark.parametrize("n", [37, 300, 1000])
def test_csv_matches_reference(R, dev, tmp_path, capfd, n):
    a = deltas(n, m=3, seed=n)
    paths = []
    for l in range(3):
        p = tmp_path / f"d{l}.csv"
        write_csv(p, perturb(a[l], l) if l != 1 else a[l], blank_every=7 if l == 2 else 0)
        paths.append(str(p))
    ref = R.load_dissimilarities(paths)
    ref_err = capfd.readouterr().err
    prob = jg.load_dissimilarities(paths, device=dev)
    ours_err = capfd.readouterr().err
    assert ours_err == ref_err and "forced to 0" in ours_err
    assert prob.modality_count() == 3 and prob.object_count() == n
    same_problem(prob, ref)


@pytest.mark.parametrize("n", [2, 129, 700])
def test_binary_matches_reference(R, dev, tmp_path, n):
    a = deltas(n, m=2, seed=100 + n)
    path = str(tmp_path / "p.jofc")
    R.save_problem_binary(a, path)  # the reference's own writer
    ref = R.load_dissimilarities([path])
    assert np.array_equal(ref, a)
    prob = jg.load_dissimilarities(path, device=dev)
    same_problem(prob, ref)


def test_binary_asymmetric_payload_averaged(R, dev, tmp_path):
    a = deltas(200, m=2, seed=7)
    b = np.stack([perturb(a[0], 1), perturb(a[1], 2)])
    path = str(tmp_path / "q.jofc")
    with open(path, "wb") as f:
        f.write(b"JOFC" + struct.pack("<4I", 1, 200, 2, 0) + b.astype("<f8").tobytes())
    ref = R.load_dissimilarities([path])
    same_problem(jg.load_dissimilarities(path, device=dev), ref)


def test_normalize_close(R, dev, tmp_path):
    a = deltas(260, m=2, seed=9)
    paths = []
    for l in range(2):
        p = tmp_path / f"n{l}.csv"
        write_csv(p, a[l])
        paths.append(str(p))
    prob = jg.load_dissimilarities(paths, device=dev, normalize=True)
    other = jg.Device(0)
    ref = jg.OmnibusProblem(list(R.load_dissimilarities(paths)), validate=False)
    x = np.random.default_rng(1).normal(size=(2, 260, 2))
    spec = jg.WeightSpec.uniform(0.5)
    s1 = jg.raw_stress(x, prob, spec, device=dev)
    s2 = jg.raw_stress(x, ref.normalized(), spec, device=other)
    assert abs(s1 - s2) <= 1e-14 * abs(s2)
    other.close()


def _bad_cases(tmp_path):
    """(name, paths) pairs; every case is rejected by the reference."""
    a = deltas(20, m=2, seed=3)
    cases = []

    def csv(name, body):
        p = tmp_path / name
        p.write_text(body)
        return str(p)

    good0 = str(tmp_path / "good0.csv")
    write_csv(good0, a[0])
    cases.append(("missing", [good0, str(tmp_path / "nope.csv")]))
    cases.append(("parse", [csv("parse.csv", "0,1\n1,abc\n")]))
    cases.append(("trailing-comma", [csv("tc.csv", "0,1,\n1,0,\n")]))
    cases.append(("ragged", [csv("ragged.csv", "0,1,2\n1,0\n2,1,0\n")]))
    cases.append(("empty", [csv("empty.csv", "\n  \n")]))
    cases.append(("nonsquare", [csv("ns.csv", "0,1,2\n1,0,1\n")]))
    cases.append(("size", [good0, csv("small.csv", "0,1\n1,0\n")]))
    b = a[1].copy()
    b[4, 7] = -2.5
    b[9, 1] = -1.0
    neg = str(tmp_path / "neg.csv")
    write_csv(neg, b)
    cases.append(("negative", [good0, neg]))
    c = a[1].copy()
    c[12, 3] = np.nan
    nan = str(tmp_path / "nan.csv")
    write_csv(nan, c)
    cases.append(("nonfinite", [nan]))
    e = a[0].copy()
    e[5, 11] *= 1.0 + 1e-6
    asym = str(tmp_path / "asym.csv")
    write_csv(asym, e)
    cases.append(("asymmetry", [good0, asym]))
    cases.append(("asym-then-parse", [asym, csv("p2.csv", "0,x\n")]))
    cases.append(("one-object", [csv("one.csv", "0\n")]))

    def raw(name, data):
        p = tmp_path / name
        p.write_bytes(data)
        return str(p)

    payload = a.astype("<f8").tobytes()
    cases.append(("magic", [raw("m.jofc", b"JOFX" + struct.pack("<4I", 1, 20, 2, 0) + payload)]))
    cases.append(("header", [raw("h.jofc", b"JOFC" + struct.pack("<2I", 1, 20))]))
    cases.append(("version", [raw("v.jofc", b"JOFC" + struct.pack("<4I", 2, 20, 2, 0) + payload)]))
    cases.append(("truncated", [raw("t.jofc", b"JOFC" + struct.pack("<4I", 1, 20, 2, 0)
                                    + payload[:-8])]))
    cases.append(("embedding", [raw("e.jofc", b"JOFC" + struct.pack("<4I", 1, 20, 2, 3)
                                    + payload[: 2 * 20 * 3 * 8])]))
    cases.append(("no-modalities", [raw("z.jofc", b"JOFC" + struct.pack("<4I", 1, 20, 0, 0))]))
    bad = a.copy()
    bad[1, 2, 3] = -1.0
    cases.append(("binary-negative", [raw("bn.jofc", b"JOFC" + struct.pack("<4I", 1, 20, 2, 0)
                                          + bad.astype("<f8").tobytes())]))
    cases.append(("no-files", []))
    return cases


def test_errors_match_reference(R, dev, tmp_path):
    for name, paths in _bad_cases(tmp_path):
        with pytest.raises(ValueError) as ref_e:
            R.load_dissimilarities(paths)
        with pytest.raises(jg.InvalidArgument) as our_e:
            jg.load_dissimilarities(paths, device=dev)
        ref_msg = ref_e.value.args[-1]
        assert str(our_e.value) == ref_msg, (name, str(our_e.value), ref_msg)


def test_resident_problem_guard(dev, tmp_path):
    a = deltas(50, m=2, seed=4)
    paths = []
    for l in range(2):
        p = tmp_path / f"g{l}.csv"
        write_csv(p, a[l])
        paths.append(str(p))
    prob = jg.load_dissimilarities(paths, device=dev)
    x = np.zeros((2, 50, 2))
    jg.raw_stress(x, prob, jg.WeightSpec.uniform(1.0), device=dev)
    # replacing the resident problem invalidates the handle
    jg.load_dissimilarities(paths, device=dev)
    with pytest.raises(jg.InvalidArgument):
        jg.raw_stress(x, prob, jg.WeightSpec.uniform(1.0), device=dev)


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_load_matches_single(tmp_path, world):
    wl = workloads.make(5, n=600)
    dense = wl.dense_delta()
    path = str(tmp_path / "s.jofc")
    with open(path, "wb") as f:
        f.write(b"JOFC" + struct.pack("<4I", 1, 600, 2, 0) + dense.astype("<f8").tobytes())
    x = wl.x0()
    single = jg.Device(0)
    ps = jg.load_dissimilarities(path, device=single)
    ref = jg.guttman_step_fast(x, ps, wl.spec, device=single)
    group = ThreadGroup(world)
    out = [None] * world
    errors = []

    def run(rank):
        try:
            d = jg.Device(0, shard=(rank, world))
            d.set_allreduce(group.hook_for(rank, "cuda:0"))
            p = jg.load_dissimilarities(path, device=d)
            out[rank] = jg.guttman_step_fast(x, p, wl.spec, device=d)
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
        np.testing.assert_allclose(out[r], ref, rtol=1e-13, atol=1e-13 * np.abs(ref).max())


def test_errors_deep_in_large_csv_match_reference(R, dev, tmp_path):
    # 2000 x 2000 CSVs (~80 MB: several 32 MB text batches, each split over the
    # host threads) with blank lines: the first bad line must be reported with
    # the reference's line number, after every row before it
    a = deltas(2000, m=1, seed=9)[0]
    rows = [",".join("%.17g" % v for v in r) for r in a]
    for name, mutate in (("parse", lambda r: r.replace(",", ",1.2.3,", 1)),
                         ("ragged", lambda r: r.rsplit(",", 1)[0])):
        for at in (1, 777, 1999):
            lines = []
            for i, r in enumerate(rows):
                if i % 7 == 3:
                    lines.append("   ")
                lines.append(mutate(r) if i == at else r)
            p = tmp_path / f"{name}_{at}.csv"
            p.write_text("\n".join(lines) + "\n")
            with pytest.raises(ValueError) as ref_e:
                R.load_dissimilarities([str(p)])
            with pytest.raises(jg.InvalidArgument) as our_e:
                jg.load_dissimilarities([str(p)], device=dev)
            assert str(our_e.value) == ref_e.value.args[-1], (name, at)
