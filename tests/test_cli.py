"""`jofc` command line (tools/jofc_cli.cpp): the parts
that run without a GPU -- `simulate` output byte-identical to the reference
library's writers, run-configuration errors identical to the reference's
parse_run_config, usage errors and exit codes."""
import os
import subprocess

import pytest

from oracle.oracle import REF_SO

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "build", "jofc")

needs_cli = pytest.mark.skipif(not os.path.exists(CLI), reason="build/jofc not built")
needs_ref = pytest.mark.skipif(not os.path.exists(REF_SO), reason="oracle/_ref not built")


def run(*args, cwd=None):
    return subprocess.run([CLI, *args], capture_output=True, text=True, cwd=cwd, timeout=120)


@pytest.fixture(scope="module")
def R():
    from oracle.oracle import Reference
    return Reference()


@needs_cli
@needs_ref
@pytest.mark.parametrize("setting,out", [("matched", "p"), ("anomaly", "q"), ("matched", "b.jofc"),
                                         ("anomaly", "c.jofc")])
def test_simulate_matches_reference_files(R, tmp_path, setting, out):
    ours, ref = tmp_path / "ours", tmp_path / "ref"
    ours.mkdir()
    ref.mkdir()
    r = run("simulate", "--setting", setting, "--n", "37", "--m", "3", "--dim", "2",
            "--n-anom", "4", "--seed", "11", "--out", str(ours / out))
    assert r.returncode == 0, r.stderr
    R.simulate_save(setting, 37, 3, 2, 4, 11, str(ref / out))
    names = sorted(os.listdir(ref))
    assert names == sorted(os.listdir(ours))
    assert len(names) >= (2 if out.endswith(".jofc") else 4)
    for name in names:
        assert (ours / name).read_bytes() == (ref / name).read_bytes(), name
    for name in names:
        assert f"wrote {ours / name}" in r.stdout


BAD_CONFIGS = {
    "no-eq": "inputs = a.csv\nw 0.5\n",
    "unknown": "inputs = a.csv\ncolour = red\n",
    "both": "inputs = a.csv\ngenerator = matched\n",
    "neither": "d = 2\n",
    "generator": "generator = other\n",
    "weight": "inputs = a.csv\nweight = fancy\n",
    "bad-u64": "inputs = a.csv\nd = -2\n",
    "bad-double": "inputs = a.csv\neps = 1e-6x\n",
    "bad-bool": "inputs = a.csv\nnormalize = maybe\n",
    "algorithm": "inputs = a.csv\nalgorithm = mds\n",
    "init": "inputs = a.csv\ninit = random\n",
    "product": "inputs = a.csv\nweight = product\n",
    "general": "inputs = a.csv\nweight = general\n",
    "matrix-missing": "inputs = a.csv\nweight = general\nweight_matrix = /nonexistent.csv\n",
}


@needs_cli
@needs_ref
@pytest.mark.parametrize("name", sorted(BAD_CONFIGS))
def test_run_config_errors_match_reference(R, tmp_path, name):
    cfg = tmp_path / f"{name}.cfg"
    cfg.write_text("# run description\n" + BAD_CONFIGS[name])
    ref_msg = R.parse_run_config(str(cfg))
    assert ref_msg is not None
    r = run("embed", "--config", str(cfg))
    assert r.returncode == 1
    assert r.stderr.strip() == f"error: {ref_msg}"


@needs_cli
def test_usage_and_exit_codes(tmp_path):
    assert run().returncode == 1
    assert run("--help").returncode == 0
    r = run("embed")
    assert r.returncode == 1 and "--config is required" in r.stderr
    r = run("embed", "--config", str(tmp_path / "missing.cfg"))
    assert r.returncode == 1 and "cannot open" in r.stderr
    r = run("frobnicate")
    assert r.returncode == 1 and "unknown command" in r.stderr
    r = run("simulate", "--setting", "matched", "--bogus", "1")
    assert r.returncode == 1 and "unknown option" in r.stderr
    r = run("simulate", "--setting", "weird")
    assert r.returncode == 1
    r = run("eval", "--embedding", "x")
    assert r.returncode == 1 and "not part of this build" in r.stderr
    cfg = tmp_path / "j.cfg"
    cfg.write_text("generator = matched\nalgorithm = jofc\n")
    r = run("embed", "--config", str(cfg))
    assert r.returncode == 1 and "not part of this build" in r.stderr
