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


def test_clock_sampler_parses_clocks_reasons_and_power():
    """The bench line's `clocks` object from nvidia-smi CSV rows (clocks, power.draw, the
    four throttle reasons, power.limit)."""
    class FakeProc:
        def terminate(self):
            pass

        def communicate(self, timeout=None):
            rows = ["1965, 1965, 310.5, 0x0, Not Active, Not Active, Not Active, Not Active, 1000.00",
                    "1792, 1965, 870.2, 0x4, Not Active, Not Active, Not Active, Active, 1000.00",
                    "1785, 1965, 990.0, 0x4, Not Active, Not Active, Not Active, Active, 1000.00",
                    "garbage"]
            return "\n".join(rows) + "\n", ""

    s = bench.ClockSampler(0)
    s.proc = FakeProc()
    out = s.stop()
    assert out["sm_mhz"] == 1792.0 and out["sm_max_mhz"] == 1965.0 and out["samples"] == 3
    assert out["reasons"] == ["sw_power_cap"]
    assert out["power_w"] == 870.2 and out["power_w_max"] == 990.0
    assert out["power_limit_w"] == 1000.0
