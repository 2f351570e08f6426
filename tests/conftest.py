import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def golden():
    return dict(np.load(GOLDEN))


def golden_spec(g, prefix, kind="oracle"):
    """Rebuild the fixture's WeightSpec for the oracle or the product API."""
    k = int(g[prefix + "kind"])
    if kind == "oracle":
        from oracle.oracle import Spec
        if k == 0:
            return Spec.uniform(float(g[prefix + "w"]))
        if k == 1:
            return Spec.general_(g[prefix + "general"])
        return Spec.product(g[prefix + "within"], float(g[prefix + "scale"]))
    from paper_1502_03391_b200 import WeightSpec
    if k == 0:
        return WeightSpec.uniform(float(g[prefix + "w"]))
    if k == 1:
        return WeightSpec.general(g[prefix + "general"])
    return WeightSpec.product(g[prefix + "within"], float(g[prefix + "scale"]))


def rel_fro(a, b):
    a, b = np.asarray(a), np.asarray(b)
    den = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (den if den > 0 else 1.0))


def rel(a, b):
    return abs(a - b) / max(abs(b), 1e-300)
