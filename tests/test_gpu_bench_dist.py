"""The torchrun path of bench.py (one process per rank, Delta sharded, the
exchange buffer all-reduced every iteration) run end to end on ONE GPU: both
ranks share the device and the collective is gloo, whose all-reduce of the
CUDA exchange buffer is staged through the host -- no kernel waits on another
rank's.  Checks the launcher plumbing the 8-GPU run uses (sharding, the
all-reduce hook, max-over-ranks timing, one JSON line from rank 0) and that the
sharded solve ends on the unsharded iterate."""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = pytest.mark.gpu


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_bench_torchrun_two_ranks_share_one_gpu():
    # (the Python all-reduce hook: NCCL, the default exchange, cannot put two
    # ranks on one GPU)
    env = dict(os.environ, JOFC_DIST_BACKEND="gloo", JOFC_BENCH_SHARE_GPU="1",
               JOFC_EXCHANGE="hook")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()),
           os.path.join(ROOT, "bench.py"), "--gpus", "2", "--config", "5", "--steps", "2",
           "--warmup", "3", "--no-cpu-baseline", "--e2e-steps", "1"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 alone prints
    out = json.loads(lines[0])
    assert out["n_gpus"] == 2
    assert out["config"]["parallelism"] == "delta-shard2"
    assert out["config"]["iterations_per_step"] == 100
    assert out["value"] > 0 and out["gpu_launches"] > 0
    # the sharded solve through the host-buffer path ends on the device-run iterate
    assert out["e2e"]["x_final_rel_diff_vs_device_run"] < 1e-12


def test_bench_oos_points_split_over_two_ranks():
    # the out-of-sample leg under torchrun: each rank embeds its half of the
    # 1000 points (independent units, no collective in the loop); rank 0 alone
    # prints the whole-batch rate (time = max over ranks)
    env = dict(os.environ, JOFC_DIST_BACKEND="gloo", JOFC_BENCH_SHARE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()),
           os.path.join(ROOT, "bench.py"), "--gpus", "2", "--oos", "--steps", "2",
           "--warmup", "3", "--no-cpu-baseline", "--e2e-steps", "1"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    out = json.loads(lines[0])
    assert out["n_gpus"] == 2 and out["value"] > 0
    assert "2 ranks" in out["config"]["parallelism"]


def test_bench_torchrun_native_nccl_one_rank():
    # the default multi-GPU exchange (the C ABI's NCCL reduce-scatter /
    # all-gather, captured in the solve) through the torchrun path: a one-rank
    # group, the only NCCL group a one-GPU box can form (NCCL refuses two
    # ranks on one device)
    env = dict(os.environ, JOFC_BENCH_NCCL_ONE_RANK="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()),
           os.path.join(ROOT, "bench.py"), "--gpus", "1", "--config", "5", "--steps", "2",
           "--warmup", "3", "--no-cpu-baseline", "--e2e-steps", "1"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    out = json.loads(lines[-1])
    assert "C-ABI NCCL" in out["config"]["collective"]
    assert out["config"]["iterations_per_step"] == 100 and out["value"] > 0
    assert out["e2e"]["x_final_rel_diff_vs_device_run"] < 1e-12


def test_bench_torchrun_falls_back_when_native_nccl_refuses():
    # the default exchange asked of a two-rank group on ONE GPU: NCCL itself
    # refuses the communicator (two ranks on one device), every rank sees
    # it, and all of them take the all-reduce hook instead -- the bench line
    # says which collective ran
    env = dict(os.environ, JOFC_DIST_BACKEND="gloo", JOFC_BENCH_SHARE_GPU="1")
    env.pop("JOFC_EXCHANGE", None)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()),
           os.path.join(ROOT, "bench.py"), "--gpus", "2", "--config", "5", "--steps", "2",
           "--warmup", "3", "--no-cpu-baseline", "--e2e-steps", "1"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    assert "C-ABI NCCL exchange unavailable" in r.stderr
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    out = json.loads(lines[0])
    assert out["n_gpus"] == 2 and out["value"] > 0
    assert "Python hook" in out["config"]["collective"]
    assert out["e2e"]["x_final_rel_diff_vs_device_run"] < 1e-12
