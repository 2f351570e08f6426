"""bench.py's reference arm (CPU): prints the same metric string as the GPU
arm, with the driver contract's keys, and maps none of the product's .so files."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def test_reference_arm_is_product_free_and_comparable():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--config", "1", "--steps", "1", "--warmup", "0",
                          "--ref-iterations", "2"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    assert line["metric"] == bench.metric_name(1, 2, 500, 2)
    assert line["config"]["workload"] == bench.workload_label(1, 2, 500, 2, 0.5, True, 100)
    assert line["product_libraries_loaded"] == []
    assert line["e2e"]["value"] == line["value"] and line["unit"] == "it/s"
    assert line["cpu_baseline"]["kind"] in ("reference", "port")
    for key in ("value", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "config"):
        assert key in line


def test_default_reference_iterations_at_least_ten():
    import argparse  # noqa: F401
    src = open(os.path.join(ROOT, "bench.py")).read()
    assert '"--ref-iterations", type=int, default=10' in src
