#!/bin/bash
# Session check: GPU suite, smoke, C3/C4 bench lines, per-pass timing (outputs in gpurun_out/r05/).
mkdir -p gpurun_out/r05
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r05/gputest.log 2>&1; echo "gputest rc=$?" >> gpurun_out/r05/gputest.log
tail -3 gpurun_out/r05/gputest.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r05/smoke.log 2>&1; tail -1 gpurun_out/r05/smoke.log
for c in 3 4; do timeout 900 python bench.py --config $c --steps 10 --warmup 3 >> gpurun_out/r05/bench.jsonl 2> gpurun_out/r05/bench_$c.err; done
timeout 600 python scripts/diag_pass.py --config 3 --modes 0 --its 19 > gpurun_out/r05/diag3.txt 2>&1
timeout 600 python scripts/diag_pass.py --config 4 --modes 0 --its 19 > gpurun_out/r05/diag4.txt 2>&1
tail -3 gpurun_out/r05/diag3.txt gpurun_out/r05/diag4.txt
python - <<'PY'
import json
for l in open("gpurun_out/r05/bench.jsonl"):
    d = json.loads(l)
    r = d.get("roofline", {})
    print(d["metric"][:70], d["value"], d["unit"], "e2e", (d.get("e2e") or {}).get("value"),
          "frac", r.get("frac"), "pass_ms", r.get("avg_launch_ms"), "cpu", (d.get("cpu_baseline") or {}).get("value"), "clk", d.get("clocks", {}).get("sm_mhz"))
PY
