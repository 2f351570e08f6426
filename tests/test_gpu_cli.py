"""`jofc embed | oos | bench` on the GPU (tools/jofc_cli.cpp, SURVEY.md 8f row
f4) against the reference library on the same files: embedding and trace
within the parity tolerances (X 1e-8 relative Frobenius, stress 1e-10)."""
import csv
import os
import subprocess

import numpy as np
import pytest

from conftest import rel_fro
from oracle.oracle import REF_SO, Spec

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "build", "jofc")

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not os.path.exists(CLI), reason="build/jofc not built"),
              pytest.mark.skipif(not os.path.exists(REF_SO), reason="oracle/_ref not built")]


def run(*args):
    return subprocess.run([CLI, *args], capture_output=True, text=True, timeout=300)


@pytest.fixture(scope="module")
def R():
    from oracle.oracle import Reference
    return Reference()


def read_embedding_csv(path):
    with open(path) as f:
        m, n, d = (int(v) for v in f.readline().split(","))
        rows = [[float(v) for v in line.split(",")] for line in f if line.strip()]
    return np.array(rows).reshape(m, n, d)


def read_trace(path):
    with open(path) as f:
        return [float(r["stress"]) for r in csv.DictReader(f)]


@pytest.mark.parametrize("init", ["averaged", "imputed"])
def test_embed_from_files_matches_reference(R, tmp_path, init):
    prefix = str(tmp_path / "sim")
    assert run("simulate", "--setting", "matched", "--n", "150", "--m", "3", "--dim", "2",
               "--seed", "5", "--out", prefix).returncode == 0
    paths = [f"{prefix}_{i}.csv" for i in (1, 2, 3)]
    cfg = tmp_path / "run.cfg"
    out = tmp_path / "emb.csv"
    cfg.write_text(f"inputs = {', '.join(paths)}\nw = 0.7\nd = 2\neps = 1e-300\n"
                   f"max_iterations = 40\ninit = {init}\nout = {out}\n")
    r = run("embed", "--config", str(cfg), "--trace", str(tmp_path / "trace.csv"))
    assert r.returncode == 0, r.stderr
    assert f"embedding: {out}" in r.stdout and "final_stress:" in r.stdout
    got = read_embedding_csv(out)
    delta = R.load_dissimilarities(paths)
    x0 = (R.averaged_procrustes_init(delta, 2) if init == "averaged"
          else R.imputed_omnibus_init(delta, 2))
    ref = R.fjofc_embed(delta, Spec.uniform(0.7), x0, 1e-300, 40)
    assert rel_fro(got, ref.x) < 1e-8, rel_fro(got, ref.x)
    trace = read_trace(tmp_path / "trace.csv")
    k = min(len(trace), len(ref.trace))
    assert max(abs(a - b) / abs(b) for a, b in zip(trace[:k], ref.trace[:k])) < 1e-10


def test_embed_generator_equals_files(tmp_path):
    # generator = matched builds Delta on the device from the same features
    prefix = str(tmp_path / "g")
    assert run("simulate", "--setting", "anomaly", "--n", "120", "--m", "2", "--dim", "2",
               "--n-anom", "5", "--seed", "9", "--out", prefix + ".jofc").returncode == 0
    common = "w = 0.5\nd = 2\neps = 1e-300\nmax_iterations = 25\n"
    (tmp_path / "a.cfg").write_text(f"inputs = {prefix}.jofc\n{common}out = {tmp_path}/a.csv\n")
    (tmp_path / "b.cfg").write_text("generator = anomaly\nn = 120\nm = 2\ndim = 2\nn_anom = 5\n"
                                    f"seed = 9\n{common}out = {tmp_path}/b.csv\n")
    for name in ("a", "b"):
        r = run("embed", "--config", str(tmp_path / f"{name}.cfg"))
        assert r.returncode == 0, r.stderr
    a = read_embedding_csv(tmp_path / "a.csv")
    b = read_embedding_csv(tmp_path / "b.csv")
    assert rel_fro(a, b) < 1e-12


def test_oos_matches_reference(R, tmp_path):
    rng = np.random.default_rng(2)
    m, n, d = 2, 80, 2
    x = rng.normal(size=(m, n, d))
    emb = tmp_path / "x.csv"
    with open(emb, "w") as f:
        f.write(f"{m},{n},{d}\n")
        for l in range(m):
            for i in range(n):
                f.write(",".join("%.17g" % v for v in x[l, i]) + "\n")
    y_true = rng.normal(size=d)
    deltas = np.stack([np.sqrt(((x[l] - y_true) ** 2).sum(1)) + 0.01 * rng.random(n)
                       for l in range(m)])
    paths = []
    for l in range(m):
        p = tmp_path / f"delta{l}.csv"
        p.write_text("\n".join("%.17g" % v for v in deltas[l]) + "\n")  # one column
        paths.append(str(p))
    r = run("oos", "--embedding", str(emb), "--deltas", *paths, "--w", "0.5", "--eps", "1e-9",
            "--max-iterations", "60", "--seed", "4", "--out", str(tmp_path / "y.csv"))
    assert r.returncode == 0, r.stderr
    assert "oos iterations:" in r.stderr
    y = np.loadtxt(tmp_path / "y.csv", delimiter=",")
    ref = R.oos_embed(x, deltas, 0.5, 1e-9, 60, 4)
    assert rel_fro(y, ref.x) < 1e-8, rel_fro(y, ref.x)


def test_bench_grid(tmp_path):
    grid = tmp_path / "grid.cfg"
    grid.write_text("n_list = 100, 160\nm_list = 2\nd = 2\nreplicates = 2\niterations = 5\n"
                    "init = averaged\nreference = true\n")
    out = tmp_path / "bench.csv"
    r = run("bench", "--grid", str(grid), "--out", str(out))
    assert r.returncode == 0, r.stderr
    assert "not part of this build" in r.stderr
    with open(out) as f:
        rows = list(csv.DictReader(f))
    assert [(r_["n"], r_["m"], r_["algorithm"]) for r_ in rows] == [("100", "2", "fjofc"),
                                                                   ("160", "2", "fjofc")]
    for r_ in rows:
        assert 0.0 < float(r_["min_step_seconds"]) <= float(r_["median_step_seconds"])
