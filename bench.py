#!/usr/bin/env python
"""bench.py -- fJOFC Guttman loop on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 3] [--impl ours|reference]

One step = one full fJOFC solve of the chosen config (BASELINE.json configs;
default config 3: m=2, n=20000, d=5, w=0.5, 100 Guttman iterations, the
config the 1/2/4/8-GPU metric is quoted on).  `value` = Guttman iterations/s
over the whole job (iterations x steps / max-over-ranks device time) with the
packed Delta resident in HBM; `e2e` = the same metric through the C ABI
(jofc_set_problem from pinned host dense Delta + jofc_fjofc_embed with host
X0/X/trace), copies inside the timed region.  Multi-GPU (torchrun): Delta's
packed tile stream is split into balanced contiguous shards; each iteration
all-reduces the m*n*d partial product (+ fidelity) with NCCL; strong scaling.

--impl reference times the reference's own CPU implementation
(oracle/_ref/libjofc_ref.so, the unmodified reference sources; the C
restatement when that was not built) on the same workload, all host threads.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIG_NAMES = {1: "C1", 2: "C2", 3: "C3", 4: "C4", 5: "C5-in"}


def metric_name(cfg, m, n, d):
    """The metric string both arms print (the driver pairs the arms by it)."""
    return f"Guttman iterations/s (fJOFC {CONFIG_NAMES[cfg]}: m={m} n={n} d={d})"


def workload_label(cfg, m, n, d, w, general_weights, iterations):
    """config.workload, the same string on both arms."""
    spec = (f"general(diag {1.0 - w:g}, off {w:g})" if general_weights else f"uniform(w={w:g})")
    return (f"{CONFIG_NAMES[cfg]} in-sample fJOFC m={m} n={n} d={d} {spec} "
            f"{iterations} Guttman iterations/solve")


def loaded_product_libraries():
    """Product .so files mapped into this process (the reference arm must map none)."""
    try:
        with open("/proc/self/maps") as f:
            maps = f.read()
    except OSError:
        return None
    return sorted({line.split()[-1] for line in maps.splitlines()
                   if "paper_1502_03391_b200" in line and line.endswith(".so")})


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def rank_device(local, torch):
    """The GPU of this rank: LOCAL_RANK (one process per GPU).  Test hook:
    JOFC_BENCH_SHARE_GPU=1 maps ranks onto the visible GPUs round-robin so the
    torchrun path runs on a 1-GPU box -- only with JOFC_DIST_BACKEND=gloo, whose
    all-reduce is host-staged (no kernel ever waits on another rank's)."""
    if os.environ.get("JOFC_BENCH_SHARE_GPU") == "1":
        return local % max(1, torch.cuda.device_count())
    return local


def init_dist(local, torch, dist):
    backend = os.environ.get("JOFC_DIST_BACKEND", "nccl")
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist.init_process_group(backend)
    return backend


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def probe_fp64(device):
    import ctypes as C
    lib = C.CDLL(os.path.join(ROOT, "paper_1502_03391_b200", "libjofc_probe.so"))
    a, b, c = C.c_double(), C.c_double(), C.c_double()
    if lib.jofc_probe_fp64(int(device), C.byref(a), C.byref(b), C.byref(c)) != 0:
        return None
    return {"dfma_tflops": a.value, "dmma_tflops": b.value, "mixed_tflops": c.value}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,"
              "power.limit")

    def __init__(self, gpu):
        self.gpu = gpu
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, smax, reasons, watts, limit = [], None, set(), [], None
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                smax = float(f[1])
            except ValueError:
                continue
            for nm, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
            try:  # board power beside the clock: a sw_power_cap run is energy-bound
                watts.append(float(f[2]))
                limit = float(f[8]) if len(f) > 8 else limit
            except ValueError:
                pass
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm),
                "power_w": float(np.median(watts)) if watts else None,
                "power_w_max": float(np.max(watts)) if watts else None,  # (power.draw lags: ~1 s average)
                "power_limit_w": limit}


def h2d_bytes_dense_upload(m, n, world, rank):
    """Bytes jofc_set_problem copies: chunks of 4 row blocks (512 rows), columns
    from the chunk's first row to n, only chunks that meet this rank's shard
    (layout: paper_1502_03391_b200/csrc/jofc_layout.h)."""
    R, C, K = 128, 64, 4
    nT = (n + C - 1) // C
    nB = (nT + 1) // 2

    def rf(B):
        return B * nT - B * (B - 1)

    bpm = rf(nB)
    from paper_1502_03391_b200 import layout
    lo, hi = layout.shard_range(m, n, rank, world)
    b = 0
    for l in range(m):
        for B0 in range(0, nB, K):
            B1 = min(nB, B0 + K)
            g0, g1 = l * bpm + rf(B0), l * bpm + rf(B1)
            if g1 <= lo or g0 >= hi:
                continue
            r0, r1 = B0 * R, min(n, B1 * R)
            if r1 > r0:
                b += (r1 - r0) * (n - r0) * 8
    return b


def oos_traffic():
    """L2 -> SM bytes per update of the persistent OOS solve (ncu; the roof is L2)."""
    path = os.path.join(ROOT, "profiles", "oos_traffic_cfg5.json")
    try:
        with open(path) as f:
            return json.load(f)["l2_to_sm_bytes_per_update"]
    except (OSError, KeyError, ValueError):
        return None


def read_traffic(cfg, kind="pass"):
    path = os.path.join(ROOT, "profiles", f"{kind}_traffic_cfg{cfg}.json")
    if os.path.exists(path):
        with open(path) as f:
            return json.load(f).get("dram_bytes_per_launch")
    return None


# --------------------------------------------------------------------- ours
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1502_03391_b200 as jg
    from paper_1502_03391_b200 import workloads
    from paper_1502_03391_b200._capi import check, dptr

    rank, world, local = env_rank()
    local = rank_device(local, torch)
    torch.cuda.set_device(local)
    backend = (init_dist(local, torch, dist)
               if world > 1 or os.environ.get("JOFC_BENCH_NCCL_ONE_RANK") == "1" else None)
    cfg = args.config
    wl = workloads.make(cfg)
    spec = wl.spec
    dev = jg.Device(local, shard=(rank, world))
    lib = dev.lib
    stream = torch.cuda.ExternalStream(dev.stream)

    # Inputs resident in HBM: Delta packed on the device from the features
    # (reference arithmetic, bit-identical to the dense host matrix), X0 on
    # the device.
    dev.upload_features(wl.in_features)
    x0_host = wl.x0()
    x0_dev = torch.from_numpy(x0_host).cuda()
    if world > 1 and args.exchange == "peer":
        # products and configuration rows through peer memory inside the
        # loop's own kernels (csrc/jofc_peer.cuh), slabs mapped by CUDA IPC
        from paper_1502_03391_b200.dist import attach_peers
        attach_peers(dev)
    elif world > 1 and args.exchange == "hook":
        from paper_1502_03391_b200.dist import attach_nccl
        attach_nccl(dev, wl.d)  # torch-owned exchange buffer, NCCL all-reduce on dev.stream
    elif world > 1 or (backend and os.environ.get("JOFC_BENCH_NCCL_ONE_RANK") == "1"):
        # the C ABI's own NCCL reduce-scatter + all-gather, in the CUDA graph
        # (JOFC_BENCH_NCCL_ONE_RANK: a one-rank group under torchrun, the test
        # hook a one-GPU box can run).  If the C ABI cannot bring NCCL up on
        # every rank (e.g. no loadable libnccl), all ranks take the Python hook
        # (torch's NCCL all-reduce) instead, and the line says so.
        from paper_1502_03391_b200.dist import attach_nccl, attach_nccl_native
        ok = 1
        try:
            attach_nccl_native(dev)
        except Exception as e:  # noqa: BLE001 (reported, then the fallback)
            print(f"[bench] C-ABI NCCL exchange unavailable on rank {rank}: {e}; "
                  f"using the all-reduce hook", file=sys.stderr)
            ok = 0
        if world > 1:
            flag = torch.tensor([ok], dtype=torch.int32, device="cuda")
            dist.all_reduce(flag, op=dist.ReduceOp.MIN)
            ok = int(flag.item())
        if not ok:
            if world > 1:
                dev.nccl_release()
                attach_nccl(dev, wl.d)
            args.exchange = "hook"

    import ctypes as C
    eps, T = 1e-300, wl.iterations
    x0_ptr = C.cast(x0_dev.data_ptr(), C.POINTER(C.c_double))

    def solve():
        check(lib.jofc_fjofc_enqueue(dev.h, C.byref(spec.c()), wl.d, x0_ptr, eps, T))

    def fetch():
        its, conv = C.c_size_t(), C.c_int()
        check(lib.jofc_fetch_result(dev.h, None, None, C.byref(its), C.byref(conv)))
        return its.value

    for _ in range(args.warmup):
        solve()
    if args.warmup > 0:
        fetch()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    barrier()
    # Large configs: CUDA events around every pass launch during the timed
    # region itself (stream launches; launch overhead is invisible at ~1 ms per
    # pass).  Small configs: the timed region replays the captured CUDA graph
    # and the pass kernel is timed with events in a separate profiled solve.
    profile_live = not args.graphs
    clocks = ClockSampler(local)
    clocks.start()
    check(lib.jofc_profile(dev.h, 1 if profile_live else 0))
    launches0 = dev.launches()
    evals0 = dev.stress_evaluations()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        solve()
    e1.record(stream)
    e1.synchronize()
    launches = dev.launches() - launches0
    x_dev = np.empty_like(x0_host)
    its_c, conv_c = C.c_size_t(), C.c_int()
    check(lib.jofc_fetch_result(dev.h, dptr(x_dev), None, C.byref(its_c), C.byref(conv_c)))
    its = its_c.value
    # iterations the device actually executed in the timed region: stress
    # evaluations counted on the device, minus sigma(X0) once per solve
    total_its = dev.stress_evaluations() - evals0 - args.steps
    pass_ms, pass_n = C.c_double(), C.c_uint64()
    if not profile_live:
        check(lib.jofc_profile(dev.h, 1))
        solve()
    check(lib.jofc_profile_read(dev.h, C.byref(pass_ms), C.byref(pass_n)))
    check(lib.jofc_profile(dev.h, 0))
    barrier()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = total_its / (ms * 1e-3)
    pairs = dev.problem_pairs()
    local_bytes = dev.problem_bytes()

    # roofline of the dominant kernel (the fused pass), from live CUDA events
    hbm_peak, hbm_src = measured_peaks()
    avg_pass_ms = pass_ms.value / max(pass_n.value, 1)
    alg_bytes = 8.0 * pairs / world  # packed Delta entries streamed per launch (this shard)
    achieved = alg_bytes / (avg_pass_ms * 1e-3) / 1e9
    fp64 = probe_fp64(local) if rank == 0 else None
    flops = (7 * wl.d + 6) * pairs / world
    roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm_peak, "unit": "GB/s",
            "frac": round(achieved / hbm_peak, 4), "traffic": read_traffic(cfg),
            "peak_source": hbm_src, "kernel": "jofc_pass_kernel",
            "algorithmic_bytes_per_launch": alg_bytes,
            "avg_launch_ms": round(avg_pass_ms, 4),
            "pass_share_of_step": (round(avg_pass_ms * (its + 1) * args.steps / ms, 4)
                                   if world == 1 else None),
            "pass_timing": "live, CUDA events around every pass launch in the timed region"
                           if profile_live else "CUDA events around every pass launch of one "
                           "extra profiled solve after the timed (graph-replay) region"}
    # Small problems on one GPU solve in ONE cooperative launch
    # (jofc_solve_persistent_kernel, kPersistentMaxBlocks in capi_internal.h):
    # the timed region holds that kernel, whose pass phase is the profiled
    # pass above; the whole-iteration rate is reported beside it.
    env_p = os.environ.get("JOFC_PERSISTENT", "")
    blocks = local_bytes // (128 * 64 * 8)
    if (world == 1 and not profile_live and env_p != "0"
            and (env_p == "1" or blocks <= 4096)):
        it_ms = ms / max(total_its, 1)
        roof["timed_region"] = ("one cooperative launch per solve: jofc_solve_persistent_kernel "
                                "(pass, grid barrier, epilogue, grid barrier per iteration)")
        roof["iteration_ms"] = round(it_ms, 5)
        roof["iteration_frac"] = round(alg_bytes / (it_ms * 1e-3) / 1e9 / hbm_peak, 4)
    if fp64:
        ach_tf = flops / (avg_pass_ms * 1e-3) / 1e12
        roof["fp64"] = {"achieved_tflops": round(ach_tf, 2),
                        "peak_tflops_dfma_measured": round(fp64["dfma_tflops"], 2),
                        "frac": round(ach_tf / fp64["dfma_tflops"], 4),
                        "algorithmic_flops_per_pair": 7 * wl.d + 6,
                        "dmma_tflops_measured": round(fp64["dmma_tflops"], 2),
                        "dfma_plus_dmma_tflops_measured": round(fp64["mixed_tflops"], 2)}
        t_h = alg_bytes / (hbm_peak * 1e9)
        t_f = flops / (fp64["dfma_tflops"] * 1e12)
        roof["roofline_ms"] = round(max(t_h, t_f) * 1e3, 4)
        roof["frac_of_roofline"] = round(max(t_h, t_f) / (avg_pass_ms * 1e-3), 4)

    # ---------------- e2e through the C ABI with pinned host buffers
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, wl, dev, spec, world, rank, torch, dist, x_dev)

    # ---------------- CPU baseline (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(wl, args)

    if rank == 0:
        line = {
            "metric": metric_name(cfg, wl.m, wl.n, wl.d),
            "value": round(value, 3), "unit": "it/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded, BASELINE.json recipe; DESIGN.md)",
            "config": {"workload": workload_label(cfg, wl.m, wl.n, wl.d, wl.w, wl.general_weights, T),
                       "iterations_per_step": its, "packed_pairs": pairs,
                       "iterations_timed": int(total_its),
                       "inputs": "packed Delta resident in HBM when the timed region starts "
                                 "(e2e: dense host Delta through the C ABI)",
                       "launch": "CUDA graph replay" if args.graphs else "stream launches",
                       "delta_bytes_resident_per_gpu": local_bytes,
                       "parallelism": f"delta-shard{world}" if world > 1 else "single",
                       "collective": (None if world == 1 and not backend else
                                      "peer memory: reduce-scatter read + mix + all-gather "
                                      "write in the loop's kernels (NVLink loads/stores)"
                                      if args.exchange == "peer" else
                                      f"{backend} all-reduce of P + fidelity per iteration "
                                      f"(Python hook)" if args.exchange == "hook" else
                                      "C-ABI NCCL per iteration: m x reduce-scatter of P row "
                                      "chunks + all-reduce of the fidelity, own-row mix, "
                                      "m x all-gather of X rows; in the CUDA graph"),
                       "l2": "inputs larger than L2 (packed Delta %.2f GB vs 126 MB L2)" % (local_bytes / 1e9)
                       if local_bytes > 126e6 * 4 else "Delta may be L2-resident"},
            "delta_entries_per_s": value * pairs,
            "delta_entries_per_s_per_gpu": value * pairs / world,
            "roofline": roof,
            "gpu_launches": int(launches),
            "clocks": clk,
        }
        if e2e:
            line["e2e"] = e2e
        if cpu:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    dev.close()
    if backend:
        dist.destroy_process_group()


def run_e2e(args, wl, dev, spec, world, rank, torch, dist, x_dev):
    """Same metric through the reference-facing C ABI with host buffers."""
    import ctypes as C

    import psutil

    from paper_1502_03391_b200._capi import _dp, check, dptr
    need = wl.m * wl.n * wl.n * 8
    if psutil.virtual_memory().available < 2.5 * need:
        return {"value": None, "unit": "it/s", "skipped": "not enough host memory for dense Delta"}
    lib = dev.lib
    delta = wl.dense_delta()  # (m, n, n) host, reference bits
    x0 = wl.x0()
    # pin the host buffers once (outside the timed region)
    cudart = torch.cuda.cudart()
    pinned = []
    for arr in (delta, x0):
        rc = cudart.cudaHostRegister(arr.ctypes.data, arr.nbytes, 0)
        pinned.append((arr, int(rc) == 0))
    x_out = np.empty_like(x0)
    trace = np.empty(wl.iterations + 1)
    x_out_pin = int(cudart.cudaHostRegister(x_out.ctypes.data, x_out.nbytes, 0)) == 0
    ptrs = (_dp * wl.m)(*[dptr(delta[l]) for l in range(wl.m)])
    its, conv = C.c_size_t(), C.c_int()
    steps = max(1, args.e2e_steps)

    split = [0.0, 0.0]  # wall seconds in the upload / the solve call

    def one():
        a = time.perf_counter()
        check(lib.jofc_set_problem(dev.h, wl.m, wl.n, ptrs, 0))
        b = time.perf_counter()
        check(lib.jofc_fjofc_embed(dev.h, C.byref(spec.c()), wl.d, dptr(x0), 1e-300,
                                   wl.iterations, dptr(x_out), dptr(trace), C.byref(its),
                                   C.byref(conv), None))
        split[0] += b - a
        split[1] += time.perf_counter() - b

    one()  # warm-up
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    split[:] = [0.0, 0.0]
    t0 = time.perf_counter()
    for _ in range(steps):
        one()
    t1 = time.perf_counter()
    sec = t1 - t0
    if world > 1:
        t = torch.tensor([sec], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        sec = float(t.item())
    h2d = h2d_bytes_dense_upload(wl.m, wl.n, world, rank) + x0.nbytes
    d2h = x_out.nbytes + 8 * (its.value + 1)
    serial = {"value": round(its.value * steps / sec, 3), "unit": "it/s",
              "ms_per_step": round(sec / steps * 1e3, 2),
              "upload_ms_per_step": round(split[0] / steps * 1e3, 2),
              "solve_ms_per_step": round(split[1] / steps * 1e3, 2),
              "path": "jofc_set_problem(pinned dense host Delta) + jofc_fjofc_embed(host X0 -> "
                      "host X, trace); wall clock, synchronous C-ABI calls, one context",
              "x_final_rel_diff_vs_device_run": float(np.linalg.norm(x_out - x_dev)
                                                      / max(np.linalg.norm(x_dev), 1e-300))}
    out = {"value": serial["value"], "unit": "it/s", "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": d2h, "steps": steps, "mode": "serial", "serial": serial,
           "x_final_rel_diff_vs_device_run": serial["x_final_rel_diff_vs_device_run"]}
    if world == 1 and not args.e2e_serial_only:
        pipe = run_e2e_pipelined(args, wl, dev, spec, delta, x0, cudart, x_dev)
        if pipe and "value" in pipe:
            out.update(value=pipe["value"], mode="double-buffered", pipelined=pipe)
            out["x_final_rel_diff_vs_device_run"] = max(out["x_final_rel_diff_vs_device_run"],
                                                        pipe["x_final_rel_diff_vs_device_run"])
        elif pipe:
            out["pipelined"] = pipe
    for arr, ok in pinned:
        if ok:
            cudart.cudaHostUnregister(arr.ctypes.data)
    if x_out_pin:
        cudart.cudaHostUnregister(x_out.ctypes.data)
    return out


def run_e2e_pipelined(args, wl, dev, spec, delta, x0, cudart, x_dev):
    """The serving form of the same public API: two contexts on the GPU,
    alternating.  Step k's host Delta upload (jofc_set_problem on one context:
    PCIe copies + pack kernels, synchronous on that context only) runs while
    step k-1's solve (jofc_fjofc_enqueue on the other context) occupies the
    SMs; step k's solve is enqueued at once, then step k-1's X and trace come
    back (jofc_fetch_result, D2H).  Every step still pays its own H2D of Delta
    and X0 and its own D2H of X and the trace inside the timed region; a step
    costs ~max(upload, solve) instead of their sum.  (Delta and X0 are the
    caller's pinned host buffers, registered by run_e2e.)"""
    import ctypes as C

    import paper_1502_03391_b200 as jg
    from paper_1502_03391_b200._capi import _dp, check, dptr
    steps = max(2, args.e2e_steps)
    try:
        other = jg.Device(dev.device)
    except Exception as e:  # noqa: BLE001 (reported in the line)
        return {"skipped": f"second context unavailable: {e}"}
    devs = [dev, other]
    lib = dev.lib
    ptrs = (_dp * wl.m)(*[dptr(delta[l]) for l in range(wl.m)])
    outs = [np.empty_like(x0) for _ in range(2)]
    traces = [np.empty(wl.iterations + 1) for _ in range(2)]
    regs = [int(cudart.cudaHostRegister(a.ctypes.data, a.nbytes, 0)) == 0 for a in outs]
    its, conv = C.c_size_t(), C.c_int()
    counted = [0]

    def upload(k):
        check(lib.jofc_set_problem(devs[k & 1].h, wl.m, wl.n, ptrs, 0))

    def enqueue(k):
        check(lib.jofc_fjofc_enqueue(devs[k & 1].h, C.byref(spec.c()), wl.d, dptr(x0), 1e-300,
                                     wl.iterations))

    def fetch(k):
        check(lib.jofc_fetch_result(devs[k & 1].h, dptr(outs[k & 1]), dptr(traces[k & 1]),
                                    C.byref(its), C.byref(conv)))
        counted[0] += its.value

    def run(n):
        upload(0)
        enqueue(0)
        for k in range(1, n):
            upload(k)    # overlaps solve k-1 on the other context
            enqueue(k)   # queued behind it: the GPU never waits for the host
            fetch(k - 1)
        fetch(n - 1)

    try:
        run(2)  # warm-up: both contexts build their graphs
        import torch
        torch.cuda.synchronize()
        counted[0] = 0
        t0 = time.perf_counter()
        run(steps)
        sec = time.perf_counter() - t0
        last = outs[(steps - 1) & 1]
        return {"value": round(counted[0] / sec, 3), "unit": "it/s", "steps": steps,
                "ms_per_step": round(sec / steps * 1e3, 2),
                "path": "two contexts alternating: jofc_set_problem(pinned dense host Delta) "
                        "of step k under the jofc_fjofc_enqueue solve of step k-1, the "
                        "enqueue of step k, then jofc_fetch_result(host X, trace) of step "
                        "k-1; wall clock",
                "x_final_rel_diff_vs_device_run": float(np.linalg.norm(last - x_dev)
                                                        / max(np.linalg.norm(x_dev), 1e-300)),
                "note": "a problem with fewer packed blocks than SMs (C1: 40 blocks, so a "
                        "40-CTA grid) also runs its solve beside the other context's on the "
                        "idle SMs, so this can exceed the one-context `value`; from C2 up "
                        "every solve fills the 148 SMs"}
    finally:
        for a, ok in zip(outs, regs):
            if ok:
                cudart.cudaHostUnregister(a.ctypes.data)
        other.close()


def cpu_baseline(wl, args):
    """The reference CPU path on this host, bounded sample of the same workload."""
    from oracle.oracle import Port, Reference, Spec
    try:
        R = Reference()
        kind = "reference"
    except (FileNotFoundError, OSError):
        R = Port()
        kind = "port"
    delta = wl.dense_delta()
    x0 = wl.x0()
    spec = (Spec.general_(wl.spec.general) if wl.general_weights else Spec.uniform(wl.w))
    cores = R.max_threads() if kind == "reference" else 1
    if kind == "reference":
        R.problem(delta)  # validated OmnibusProblem, outside the timing
    t0 = time.perf_counter()
    R.fjofc_embed(delta, spec, x0, 1e-300, 1, parallel=True)
    t1 = time.perf_counter() - t0
    n_it = int(max(1, min(wl.iterations, args.cpu_seconds / max(t1, 1e-9))))
    t0 = time.perf_counter()
    r = R.fjofc_embed(delta, spec, x0, 1e-300, n_it, parallel=True)
    sec = time.perf_counter() - t0
    its = r.iterations
    out = {"value": round(its / sec, 5), "unit": "it/s", "cores": cores, "kind": kind,
           "sample": f"{its} Guttman iterations of fjofc_embed on the full "
                     f"{CONFIG_NAMES[wl.cfg]} workload (parallel=true, OpenMP), call "
                     f"wall time incl. sigma(X0)",
           "seconds": round(sec, 3)}
    if kind == "reference":
        R.release()
    return out


# ------------------------------------------------------------- reference arm
def run_reference(args):
    """The reference's own CPU implementation (oracle/_ref: the unmodified
    reference sources; the C restatement when _ref was not built) on the same
    workload, all host threads.  Inputs come from the reference's own Rng and
    euclidean_distance_matrix (oracle/workloads_ref.py, bit-identical to the
    product generator): this arm loads nothing of the product package."""
    rank, world, _ = env_rank()
    if rank != 0:
        return
    from oracle import workloads_ref
    from oracle.oracle import Reference
    cfg = args.config
    wl = workloads_ref.make(cfg)
    R = wl.impl
    kind = "reference" if isinstance(R, Reference) else "port"
    delta = wl.dense_delta()
    x0 = wl.x0()
    spec = wl.spec
    cores = R.max_threads() if kind == "reference" else 1
    if kind == "reference":
        R.problem(delta)  # validated OmnibusProblem, outside the timing
    per_step = args.ref_iterations
    for _ in range(args.warmup):
        R.fjofc_embed(delta, spec, x0, 1e-300, per_step, parallel=True)
    t0 = time.perf_counter()
    total = 0
    for _ in range(args.steps):
        total += R.fjofc_embed(delta, spec, x0, 1e-300, per_step, parallel=True).iterations
    sec = time.perf_counter() - t0
    value = total / sec
    line = {
        "impl": "reference",
        "metric": metric_name(cfg, wl.m, wl.n, wl.d),
        "value": round(value, 5), "unit": "it/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(sec / args.steps * 1e3, 2),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded, BASELINE.json recipe; DESIGN.md)",
        "config": {"workload": workload_label(cfg, wl.m, wl.n, wl.d, wl.w, wl.general_weights,
                                             wl.iterations),
                   "iterations_per_step": per_step,
                   "inputs": "dense host Delta (reference OmnibusProblem), reference Rng X0"},
        "delta_entries_per_s": value * wl.m * wl.n * (wl.n - 1) / 2,
        "cpu_baseline": {"value": round(value, 5), "unit": "it/s", "cores": cores, "kind": kind,
                         "sample": f"{per_step} Guttman iterations of fjofc_embed per step on "
                                   f"the full {CONFIG_NAMES[cfg]} workload, parallel=true "
                                   f"(OpenMP, {cores} threads); sigma(X0) once per step"},
        "e2e": {"value": round(value, 5), "unit": "it/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "product_libraries_loaded": loaded_product_libraries(),
    }
    if kind == "reference":
        R.release()
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------ out-of-sample
def run_oos(args):
    """C5 out-of-sample: k = 1000 new objects embedded against the frozen
    in-sample configuration, batched, 100 fixed Guttman updates per step.
    Under torchrun the points are split over the ranks (independent units,
    SURVEY.md 8e: no collective in the loop); time = max over ranks."""
    import ctypes as C

    import torch

    import paper_1502_03391_b200 as jg
    from paper_1502_03391_b200 import workloads
    from paper_1502_03391_b200._capi import check, dptr

    import torch.distributed as dist

    rank, world, local = env_rank()
    local = rank_device(local, torch)
    torch.cuda.set_device(local)
    if world > 1:
        init_dist(local, torch, dist)

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    wl = workloads.make(5)
    dev = jg.Device(local)
    lib = dev.lib
    # in-sample embedding (100 iterations on the GPU, the C5 recipe)
    dev.upload_features(wl.in_features)
    x0 = wl.x0()
    xin = np.empty_like(x0)
    check(lib.jofc_fjofc_enqueue(dev.h, C.byref(wl.spec.c()), wl.d, dptr(x0), 1e-300,
                                 wl.iterations))
    its = C.c_size_t()
    conv = C.c_int()
    check(lib.jofc_fetch_result(dev.h, dptr(xin), None, C.byref(its), C.byref(conv)))
    k_all, m, n, d, T = wl.oos_points, wl.m, wl.n, wl.d, 100
    q_lo, q_hi = k_all * rank // world, k_all * (rank + 1) // world  # this rank's points
    k = q_hi - q_lo
    od = np.ascontiguousarray(wl.oos_deltas()[q_lo:q_hi])
    y0 = np.stack([jg.oos_start(xin, workloads.OOS_SEED + q) for q in range(q_lo, q_hi)])
    xs = torch.from_numpy(xin).cuda()
    ods = torch.from_numpy(od).cuda()
    y0s = torch.from_numpy(y0).cuda()
    yout = torch.empty_like(y0s)
    P = C.POINTER(C.c_double)

    def cast(t):
        return C.cast(t.data_ptr(), P)

    def step():
        check(lib.jofc_oos_batch(dev.h, k, m, n, d, cast(xs), cast(ods), wl.w, cast(y0s), 1e-300,
                                 T, 1, cast(yout), None, None))

    for _ in range(args.warmup):
        step()
    barrier()
    launches0 = dev.launches()
    clocks = ClockSampler(local)
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    stream = torch.cuda.ExternalStream(dev.stream)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    e1.synchronize()
    sec = max_over_ranks(e0.elapsed_time(e1) * 1e-3)
    barrier()
    clk = clocks.stop()
    launches = dev.launches() - launches0
    value = T * args.steps / sec
    # e2e: host buffers through the C ABI (H2D of deltas, X, y0 and D2H of y
    # every step); the host buffers are page-locked once, outside the timed
    # region, as the in-sample e2e does
    yh = np.empty_like(y0)
    cudart = torch.cuda.cudart()
    pinned = [arr for arr in (od, xin, y0, yh)
              if int(cudart.cudaHostRegister(arr.ctypes.data, arr.nbytes, 0)) == 0]
    check(lib.jofc_oos_batch(dev.h, k, m, n, d, dptr(xin), dptr(od), wl.w, dptr(y0), 1e-300,
                             T, 1, dptr(yh), None, None))  # warm-up
    barrier()
    t0 = time.perf_counter()
    e2e_steps = max(1, args.e2e_steps)
    for _ in range(e2e_steps):
        check(lib.jofc_oos_batch(dev.h, k, m, n, d, dptr(xin), dptr(od), wl.w, dptr(y0), 1e-300,
                                 T, 1, dptr(yh), None, None))
    e2e = T * e2e_steps / max_over_ranks(time.perf_counter() - t0)
    e2e_serial = e2e
    e2e_pipe = None
    if world == 1 and not args.e2e_serial_only:
        # serving form: two contexts, one host thread each (ctypes drops the
        # GIL), so one batch's PCIe copies run under the other's solve; every
        # batch still pays its own H2D of deltas/X/y0 and D2H of y
        import threading
        other = jg.Device(local)
        yh2 = np.empty_like(y0)
        ok2 = int(cudart.cudaHostRegister(yh2.ctypes.data, yh2.nbytes, 0)) == 0
        n_each = max(1, e2e_steps // 2)
        errs = []

        def worker(dv, yb, n_steps):
            try:
                for _ in range(n_steps):
                    check(lib.jofc_oos_batch(dv.h, k, m, n, d, dptr(xin), dptr(od), wl.w,
                                             dptr(y0), 1e-300, T, 1, dptr(yb), None, None))
            except Exception as e:  # noqa: BLE001 (re-raised below)
                errs.append(e)

        worker(other, yh2, 1)  # warm-up of the second context
        t0 = time.perf_counter()
        ths = [threading.Thread(target=worker, args=(dv, yb, n_each))
               for dv, yb in ((dev, yh), (other, yh2))]
        for th in ths:
            th.start()
        for th in ths:
            th.join()
        psec = time.perf_counter() - t0
        if errs:
            raise errs[0]
        e2e_pipe = {"value": round(T * 2 * n_each / psec, 2), "unit": "batch-it/s",
                    "steps": 2 * n_each,
                    "path": "two contexts, one host thread each, jofc_oos_batch with host "
                            "buffers; one batch's copies overlap the other's solve; wall clock",
                    "y_max_abs_diff_between_contexts": float(np.max(np.abs(yh - yh2)))}
        e2e = e2e_pipe["value"]
        if ok2:
            cudart.cudaHostUnregister(yh2.ctypes.data)
        other.close()
    for arr in pinned:
        cudart.cudaHostUnregister(arr.ctypes.data)
    hbm_peak, hbm_src = measured_peaks()
    bytes_per_it = od.nbytes
    if rank != 0:
        dev.close()
        return
    # the roofs of an L2-resident update: delta bytes at the measured L2 read
    # bandwidth of a working set this size, and the algorithmic FP64 work
    # (5d + 7 flops per delta entry) at the measured DFMA peak
    import ctypes as C2
    probe = C2.CDLL(os.path.join(ROOT, "paper_1502_03391_b200", "libjofc_probe.so"))
    l2 = C2.c_double()
    l2_ok = probe.jofc_probe_l2_read(int(local), C2.c_size_t(bytes_per_it), C2.byref(l2)) == 0
    fp64 = probe_fp64(local)
    it_s = sec / (T * args.steps)
    entries = od.size
    t_l2 = bytes_per_it / (l2.value * 1e9) if l2_ok else None
    t_fp = entries * (5 * d + 7) / (fp64["dfma_tflops"] * 1e12) if fp64 else None
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        from oracle.oracle import Port, Reference
        try:
            R, kind = Reference(), "reference"
        except (FileNotFoundError, OSError):
            R, kind = Port(), "port"
        sample = k  # the whole batch (~1 s of 16-thread CPU work)
        t0 = time.perf_counter()
        R.oos_batch(xin, od[:sample], wl.w, y0[:sample], 1e-300, T, fixed=True)
        csec = time.perf_counter() - t0
        cpu = {"value": round(T * sample / k_all / csec, 4), "unit": "batch-it/s", "kind": kind,
               "cores": R.max_threads() if kind == "reference" else os.cpu_count(),
               "sample": f"{sample} of {k} points x {T} oos_step_fast+oos_stress "
                         f"(reference functions, OpenMP over points), scaled to the batch",
               "seconds": round(csec, 3)}
    line = {
        "metric": f"OOS Guttman iterations/s of a {k_all}-point batch (fJOFC C5: m={m} n={n} d={d})",
        "value": round(value, 2), "unit": "batch-it/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(sec / args.steps * 1e3, 3),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded, BASELINE.json recipe; DESIGN.md)",
        "config": {"workload": f"C5-OOS k={k_all} new objects, {T} fixed updates/step, "
                               f"X from a 100-iteration GPU in-sample solve",
                   "parallelism": (f"points split over {world} ranks, no collective in the "
                                   f"loop" if world > 1 else "single"),
                   "l2": "delta rows 80 MB fit in the 126 MB L2 (re-read every update)"},
        "point_iterations_per_s": round(value * k_all, 1),
        "roofline": {"bound": "l2", "achieved": round(bytes_per_it / it_s / 1e9, 1),
                     "peak": round(l2.value, 1) if l2_ok else None, "unit": "GB/s",
                     "frac": round(bytes_per_it / it_s / 1e9 / l2.value, 4) if l2_ok else None,
                     "traffic": oos_traffic(),
                     "peak_source": f"measured here: L2-resident reads of a {bytes_per_it / 1e6:.0f} "
                                    f"MB buffer (libjofc_probe.so jofc_probe_l2_read)",
                     "per": "rank 0's GPU (its share of the delta rows)",
                     "kernel": ("jofc_oos_solve_kernel: the whole batch solve in one launch "
                                "(+ jofc_oos_permute_kernel once per batch); update_us = step "
                                "time / updates"),
                     "update_us": round(it_s * 1e6, 2),
                     "fp64": ({"algorithmic_flops_per_entry": 5 * d + 7,
                               "achieved_tflops": round(entries * (5 * d + 7) / it_s / 1e12, 2),
                               "peak_tflops_dfma_measured": round(fp64["dfma_tflops"], 2),
                               "frac": round(t_fp / it_s, 4)} if fp64 else None),
                     "roofline_us": (round(max(t_l2, t_fp) * 1e6, 2)
                                     if t_l2 is not None and t_fp is not None else None),
                     "frac_of_roofline": (round(max(t_l2, t_fp) / it_s, 4)
                                          if t_l2 is not None and t_fp is not None else None),
                     "hbm_peak_gbs": hbm_peak,
                     "note": "delta rows (80 MB) stay in the 126 MB L2 across updates: the roof "
                             "is the slower of L2 reads and FP64 work, not HBM"},
        "gpu_launches": int(launches), "clocks": clk,
        "e2e": {"value": round(e2e, 2), "unit": "batch-it/s",
                "h2d_bytes_per_step": int(od.nbytes + xin.nbytes + y0.nbytes),
                "d2h_bytes_per_step": int(yh.nbytes),
                "mode": "double-buffered" if e2e_pipe else "serial",
                "serial": {"value": round(e2e_serial, 2), "unit": "batch-it/s",
                           "path": "one context, jofc_oos_batch with host buffers back to back; "
                                   "wall clock"},
                **({"pipelined": e2e_pipe} if e2e_pipe else {})},
    }
    if cpu:
        line["cpu_baseline"] = cpu
    print(json.dumps(line), flush=True)
    dev.close()


def run_init(args):
    """the reference's default initialiser
    (averaged_procrustes_init, proj/src/init.cpp:57-88) on the resident Delta.
    One step = one whole init (m + 1 cMDS subspace iterations + Procrustes)."""
    import ctypes as C

    import torch

    import paper_1502_03391_b200 as jg
    from paper_1502_03391_b200 import workloads
    from paper_1502_03391_b200._capi import check, dptr

    rank, world, local = env_rank()
    if rank != 0:
        return
    torch.cuda.set_device(local)
    wl = workloads.make(args.config)
    m, n, d = wl.m, wl.n, wl.d
    dev = jg.Device(local)
    lib = dev.lib
    dev.upload_features(wl.in_features)
    out = np.empty((m, n, d))

    def step():
        check(lib.jofc_init_averaged_procrustes(dev.h, d, dptr(out)))

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    launches0 = dev.launches()
    check(lib.jofc_profile(dev.h, 1))
    clocks = ClockSampler(local)
    clocks.start()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    torch.cuda.synchronize()
    sec = time.perf_counter() - t0
    clk = clocks.stop()
    launches = dev.launches() - launches0
    mv_ms, mv_n = C.c_double(), C.c_uint64()
    check(lib.jofc_profile_read(dev.h, C.byref(mv_ms), C.byref(mv_n)))
    check(lib.jofc_profile(dev.h, 0))
    sweeps = mv_n.value / args.steps
    mv_share = mv_ms.value / (sec * 1e3)
    mv_avg_ms = mv_ms.value / max(1, mv_n.value)
    s_bytes = n * n * 8  # the dense double-centred S streamed once per sweep
    achieved = s_bytes / (mv_avg_ms * 1e-3) / 1e9
    hbm_peak, hbm_src = measured_peaks()
    # e2e: host Delta through the public API (dense H2D + pack, init, D2H of X)
    e2e = None
    delta = wl.dense_delta() if not (args.no_e2e and args.no_cpu_baseline) else None
    if not args.no_e2e:
        mods = list(delta)
        # the host Delta page-locked once outside the timed region, as the
        # in-sample e2e does
        cudart = torch.cuda.cudart()
        pinned = int(cudart.cudaHostRegister(delta.ctypes.data, delta.nbytes, 0)) == 0
        e2e_steps = max(1, args.e2e_steps)
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            prob = jg.OmnibusProblem(mods, validate=False)
            jg.averaged_procrustes_init(prob, d, device=dev)
        e2e_sec = (time.perf_counter() - t0) / e2e_steps
        if pinned:
            cudart.cudaHostUnregister(delta.ctypes.data)
        e2e = {"value": round(1.0 / e2e_sec, 4), "unit": "inits/s",
               "h2d_bytes_per_step": h2d_bytes_dense_upload(m, n, 1, 0),
               "d2h_bytes_per_step": int(out.nbytes),
               "path": "OmnibusProblem(host Delta) -> averaged_procrustes_init (upload of the "
                       "upper part + the whole init + X back)"}
    cpu = None
    if not args.no_cpu_baseline:
        from oracle.oracle import Port, Reference
        try:
            R = Reference()
        except (FileNotFoundError, OSError):
            R = None
        if R is not None:
            R.problem(delta)
            # bounded sample: the cMDS of the modality average, one of the m + 1
            # eigen-solves of the init, timed whole; its sweep count is the GPU's
            # (same iteration, same start)
            check(lib.jofc_profile(dev.h, 1))
            xa = np.empty((n, d))
            check(lib.jofc_cmds(dev.h, -1, d, dptr(xa)))
            check(lib.jofc_profile_read(dev.h, C.byref(mv_ms), C.byref(mv_n)))
            check(lib.jofc_profile(dev.h, 0))
            t0 = time.perf_counter()
            R.cmds(delta, -1, d)
            csec = time.perf_counter() - t0
            cpu = {"value": round(mv_n.value / csec, 3), "unit": "sweeps/s", "kind": "reference",
                   "cores": R.max_threads(),
                   "sample": f"jofc_ref::cmds of the modality average ({mv_n.value} subspace "
                             f"sweeps at n={n}, p={d + 4}; OpenMP), call wall time",
                   "seconds": round(csec, 3)}
            R.release()
    line = {
        "metric": f"averaged_procrustes_init (fJOFC default init) per second, "
                  f"{CONFIG_NAMES[wl.cfg]}",
        "value": round(args.steps / sec, 4), "unit": "inits/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(sec / args.steps * 1e3, 3), "higher_is_better": True,
        "scaling": "replicas only", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded, BASELINE.json recipe; DESIGN.md)",
        "config": {"workload": f"{CONFIG_NAMES[wl.cfg]} init: m+1={m + 1} cMDS eigen-solves "
                               f"(shifted subspace iteration, p={d + 4}) + Procrustes",
                   "l2": f"S is {s_bytes / 1e9:.2f} GB per solve, larger than L2"},
        "sweeps_per_s": round(sweeps * args.steps / sec, 1), "sweeps_per_init": sweeps,
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm_peak,
                     "unit": "GB/s", "frac": round(achieved / hbm_peak, 4),
                     "traffic": read_traffic(wl.cfg, "init"),
                     "peak_source": hbm_src, "kernel": "matvec_sym_kernel (S Q)",
                     "kernel_ms": round(mv_avg_ms, 4),
                     "share_of_step": round(mv_share, 4)},
        "gpu_launches": int(launches), "clocks": clk,
    }
    if e2e:
        line["e2e"] = e2e
    if cpu:
        line["cpu_baseline"] = cpu
        line["sweeps_per_s_vs_cpu"] = round(line["sweeps_per_s"] / cpu["value"], 1)
    print(json.dumps(line), flush=True)
    dev.close()


def run_ingest(args):
    """load_dissimilarities from a .jofc problem file
    straight into the packed device layout (jofc_load_problem_files), against
    the reference's load_dissimilarities on the same file.  The file sits in
    /dev/shm (page cache), so the pipeline, not the disk, is measured."""
    import ctypes as C
    import shutil
    import struct
    import tempfile

    import torch

    import paper_1502_03391_b200 as jg
    from paper_1502_03391_b200 import workloads

    rank, world, local = env_rank()
    if rank != 0:
        return
    torch.cuda.set_device(local)
    wl = workloads.make(args.config)
    m, n = wl.m, wl.n
    root = "/dev/shm" if os.path.isdir("/dev/shm") else None
    tmp = tempfile.mkdtemp(prefix="jofc_ingest_", dir=root)
    try:
        path = os.path.join(tmp, "problem.jofc")
        dense = wl.dense_delta()
        with open(path, "wb") as f:
            f.write(b"JOFC" + struct.pack("<4I", 1, n, m, 0))
            for l in range(m):
                f.write(np.ascontiguousarray(dense[l], dtype="<f8").tobytes())
        nbytes = os.path.getsize(path)
        dev = jg.Device(local)
        for _ in range(args.warmup):
            jg.load_dissimilarities(path, device=dev)
        torch.cuda.synchronize()
        launches0 = dev.launches()
        clocks = ClockSampler(local)
        clocks.start()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            jg.load_dissimilarities(path, device=dev)
        torch.cuda.synchronize()
        sec = time.perf_counter() - t0
        clk = clocks.stop()
        launches = dev.launches() - launches0
        gbs = nbytes * args.steps / sec / 1e9
        # pinned host -> device copy bandwidth on this box (the link the panels cross)
        hbuf = torch.empty(1 << 28, dtype=torch.uint8, pin_memory=True)
        dbuf = torch.empty(1 << 28, dtype=torch.uint8, device="cuda")
        for _ in range(3):
            dbuf.copy_(hbuf, non_blocking=True)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            dbuf.copy_(hbuf, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        h2d = 10 * (1 << 28) / (e0.elapsed_time(e1) * 1e-3) / 1e9
        del hbuf, dbuf
        cpu = None
        if not args.no_cpu_baseline:
            from oracle.oracle import Reference
            try:
                R = Reference()
            except (FileNotFoundError, OSError):
                R = None
            if R is not None:
                t0 = time.perf_counter()
                R.load_dissimilarities([path])
                csec = time.perf_counter() - t0
                cpu = {"value": round(nbytes / csec / 1e9, 3), "unit": "GB/s", "kind": "reference",
                       "cores": 1, "sample": f"jofc_ref::load_dissimilarities of the same "
                                             f"{nbytes / 1e9:.2f} GB .jofc file (host dense "
                                             f"problem, validated), one call",
                       "seconds": round(csec, 3)}
        dev.close()
    finally:
        shutil.rmtree(tmp, ignore_errors=True)
    line = {
        "metric": f"load_dissimilarities (.jofc -> packed HBM layout) GB/s of file payload, "
                  f"{CONFIG_NAMES[wl.cfg]}",
        "value": round(gbs, 3), "unit": "GB/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(sec / args.steps * 1e3, 3),
        "higher_is_better": True, "scaling": "replicas only", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded, BASELINE.json recipe; DESIGN.md)",
        "config": {"workload": f"{CONFIG_NAMES[wl.cfg]} problem file m={m} n={n} "
                               f"({nbytes / 1e9:.2f} GB) in /dev/shm",
                   "l2": "file payload streamed once through pinned panels"},
        "roofline": {"bound": "h2d", "achieved": round(gbs, 2), "peak": round(h2d, 1),
                     "unit": "GB/s", "frac": round(gbs / h2d, 4), "traffic": None,
                     "peak_source": "measured here: pinned 256 MiB host->device copies",
                     "kernel": "jofc_pack_kernel + jofc_ingest_combine_kernel pipeline"},
        "gpu_launches": int(launches), "clocks": clk,
        "e2e": {"value": round(gbs, 3), "unit": "GB/s", "h2d_bytes_per_step": int(nbytes),
                "d2h_bytes_per_step": 8 * m},
    }
    if cpu:
        line["cpu_baseline"] = cpu
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=3, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-serial-only", action="store_true",
                    help="e2e: one context, upload and solve back to back (no double buffering)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--ref-iterations", type=int, default=10)
    ap.add_argument("--oos", action="store_true", help="C5 out-of-sample batch (config 5)")
    ap.add_argument("--init", action="store_true",
                    help="averaged_procrustes_init on the resident Delta (SURVEY 8f row f1)")
    ap.add_argument("--ingest", action="store_true",
                    help="stream a .jofc problem file into the device layout (SURVEY 8f row f2)")
    ap.add_argument("--exchange", default=os.environ.get("JOFC_EXCHANGE", "nccl"),
                    choices=["nccl", "hook", "peer"],
                    help="multi-GPU exchange: the C ABI's NCCL reduce-scatter/all-gather "
                         "(default), a Python all-reduce hook, or peer-memory kernels")
    ap.add_argument("--graphs", type=int, default=None,
                    help="replay CUDA graphs in the timed region (default: on for configs 1,2,5)")
    args = ap.parse_args()
    if args.graphs is None:
        args.graphs = args.config in (1, 2, 5)
    if args.warmup < 3:
        print("warning: fewer than 3 warm-up steps", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args)
    elif args.oos:
        run_oos(args)
    elif args.init:
        run_init(args)
    elif args.ingest:
        run_ingest(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
