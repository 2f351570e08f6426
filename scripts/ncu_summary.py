"""Summarise an ncu report (or a launch-list CSV) into profiles/.

python scripts/ncu_summary.py report.ncu-rep out.json [--pairs P --bytes B]
python scripts/ncu_summary.py --launches launches.csv out.json
"""
import argparse
import collections
import csv
import io
import json
import subprocess


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    kernels = []
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))
        u = dict(zip(hdr, units))
        kernels.append((d, u))
    return kernels


def num(s):
    try:
        return float(str(s).replace(",", ""))
    except ValueError:
        return None


KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]


def summarize_rep(rep):
    res = []
    for d, u in raw_metrics(rep):
        k = {"kernel": d.get("Kernel Name"), "id": d.get("ID")}
        for key in KEYS:
            if key in d:
                k[key] = {"value": num(d[key]), "unit": u.get(key)}
        res.append(k)
    return res


def stall_breakdown(rep):
    """Warp-state samples by reason and by SASS opcode (ncu source page)."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    by_reason, by_op = collections.Counter(), collections.defaultdict(collections.Counter)
    total = 0
    instrs = 0
    for r in rows[2:]:
        if len(r) < len(hdr):
            continue
        src = r[idx["Source"]].strip().split()
        op = (src[1] if src and src[0].startswith("@") else (src[0] if src else "")).split(".")[0]
        total += int(r[idx["# Samples"]] or 0)
        instrs += int(r[idx["Instructions Executed"]] or 0)
        for h in cols:
            v = int(r[idx[h]] or 0)
            by_reason[h[6:]] += v
            by_op[op][h[6:]] += v
    ops = sorted(by_op, key=lambda o: -sum(by_op[o].values()))[:12]
    return {"samples": total, "warp_instructions": instrs,
            "by_reason": {k: round(v / total, 4) for k, v in by_reason.most_common()},
            "by_opcode": {o: {"share": round(sum(by_op[o].values()) / total, 4),
                              "top": dict(by_op[o].most_common(3))} for o in ops}}


def summarize_launches(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    idx = {h: i for i, h in enumerate(hdr)}
    per = collections.defaultdict(list)
    for r in rows[start + 1:]:
        if len(r) < len(hdr) or r[idx["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = r[idx["Kernel Name"]].split("(")[0]
        v = num(r[idx["Metric Value"]])
        unit = r[idx["Metric Unit"]]
        scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(unit, 1.0)
        per[name].append(v * scale)
    total = sum(sum(v) for v in per.values())
    return {name: {"launches": len(v), "total_us": round(sum(v), 2),
                   "avg_us": round(sum(v) / len(v), 3), "share": round(sum(v) / total, 4)}
            for name, v in sorted(per.items(), key=lambda kv: -sum(kv[1]))}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("src")
    ap.add_argument("out")
    ap.add_argument("--launches", action="store_true")
    ap.add_argument("--note", default="")
    ap.add_argument("--stalls", action="store_true", help="add the source-page stall breakdown")
    a = ap.parse_args()
    data = summarize_launches(a.src) if a.launches else summarize_rep(a.src)
    if a.stalls and not a.launches:
        data = {"kernels": data, "stalls": stall_breakdown(a.src)}
    with open(a.out, "w") as f:
        json.dump({"source": a.src, "note": a.note, "data": data}, f, indent=1)
    print(json.dumps(data, indent=1)[:3000])


if __name__ == "__main__":
    main()
