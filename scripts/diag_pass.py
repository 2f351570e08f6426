"""Time the fused pass kernel alone under experiment switches (JOFC_DIAG).

python scripts/diag_pass.py [--config 3] [--modes 0,1,2,3]
Modes (results are WRONG for modes != 0; timing experiments only):
  0 normal, 1 no column RED, 2 column plain stores, 3 no column reduction.
"""
import argparse
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1502_03391_b200 as jg  # noqa: E402
from paper_1502_03391_b200 import workloads  # noqa: E402
from paper_1502_03391_b200._capi import check, dptr  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--modes", default="0,1,2,3")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--its", type=int, default=0,
                    help="iterations per solve (0: single-pass solves; >0 times every pass of "
                         "real solves: iteration 0 per-pair fidelity, later ones identity form)")
    a = ap.parse_args()
    modes = [int(x) for x in a.modes.split(",")]
    if len(modes) > 1 or os.environ.get("JOFC_DIAG", str(modes[0])) != str(modes[0]):
        # the library reads JOFC_DIAG once per process: one process per mode
        import subprocess
        for mode in modes:
            argv = [sys.executable, os.path.abspath(__file__), "--config", str(a.config),
                    "--modes", str(mode), "--iters", str(a.iters), "--its", str(a.its)]
            if a.n:
                argv += ["--n", str(a.n)]
            subprocess.run(argv, env=dict(os.environ, JOFC_DIAG=str(mode)), check=True)
        return
    wl = workloads.make(a.config, n=a.n)
    dev = jg.Device(0)
    dev.upload_features(wl.in_features)
    x0 = wl.x0()
    lib = dev.lib
    pairs = dev.problem_pairs()
    for mode in modes:
        # single-pass solves (max_it = 0): every launch does the full pass even
        # when the experiment corrupts the iterate
        for rep in range(2):
            check(lib.jofc_profile(dev.h, 1))
            for _ in range(max(1, a.iters // (a.its + 1))):
                check(lib.jofc_fjofc_enqueue(dev.h, C.byref(wl.spec.c()), wl.d, dptr(x0), 1e-300,
                                             a.its))
            ms, n = C.c_double(), C.c_uint64()
            check(lib.jofc_profile_read(dev.h, C.byref(ms), C.byref(n)))
        avg = ms.value / n.value
        print(f"cfg{a.config} mode {mode}: pass {avg:.4f} ms  {8 * pairs / avg / 1e6:.1f} GB/s "
              f"({n.value} launches)", flush=True)


if __name__ == "__main__":
    main()
