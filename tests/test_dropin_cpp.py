"""The C++ drop-in (include/jofc/*.hpp -> libjofc.so -> C ABI -> CUDA) run
through tests/cpp/dropin_parity.cpp, a reference-style parity suite."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "build", "dropin_parity")


def _build():
    if not os.path.exists(BIN):
        subprocess.run(["make", "-C", ROOT, "build/dropin_parity"], check=True)


def test_dropin_library_exports_reference_api():
    _build()
    out = subprocess.run(["nm", "-DC", "--defined-only",
                          os.path.join(ROOT, "paper_1502_03391_b200", "libjofc.so")],
                         capture_output=True, text=True, check=True).stdout
    for sym in ("jofc::fjofc_embed(jofc::OmnibusProblem const&, jofc::WeightSpec const&, "
                "jofc::SolveOptions const&)",
                "jofc::guttman_step_fast(jofc::Configuration const&, jofc::OmnibusProblem const&, "
                "jofc::WeightSpec const&, bool)",
                "jofc::raw_stress(jofc::Configuration const&, jofc::OmnibusProblem const&, "
                "jofc::WeightSpec const&, bool)",
                "jofc::oos_embed(jofc::Configuration const&, jofc::OosDissimilarity const&, double, "
                "jofc::OosOptions const&, unsigned long)",
                "jofc::oos_step_fast(jofc::DenseMatrix const&, jofc::Configuration const&, "
                "jofc::OosDissimilarity const&, double)",
                "jofc::oos_stress(jofc::DenseMatrix const&, jofc::Configuration const&, "
                "jofc::OosDissimilarity const&, double)",
                "jofc::stress_pair_count(unsigned long, unsigned long)"):
        assert sym in out, sym


@pytest.mark.gpu
def test_dropin_cpp_parity_suite():
    _build()
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=900)
    print(r.stdout, r.stderr[-4000:])
    assert r.returncode == 0, r.stderr[-4000:]
    assert "0 failures" in r.stdout
