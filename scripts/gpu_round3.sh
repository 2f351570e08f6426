#!/bin/bash
# Round-3 bench sweep on one box: every config's bench line, the OOS leg,
# the reference arm, init / ingest legs (outputs in gpurun_out/r03/).
mkdir -p gpurun_out/r03
: > gpurun_out/r03/bench_all.jsonl
for c in 3 4 1 2 5; do timeout 900 python bench.py --config $c --steps 10 --warmup 3 >> gpurun_out/r03/bench_all.jsonl 2> gpurun_out/r03/bench_$c.err; done
timeout 600 python bench.py --oos --steps 10 --warmup 3 >> gpurun_out/r03/bench_all.jsonl 2>> gpurun_out/r03/bench_oos.err
timeout 900 python bench.py --init --config 3 --steps 3 --warmup 3 --no-cpu-baseline >> gpurun_out/r03/bench_all.jsonl 2>> gpurun_out/r03/init.err
timeout 600 python bench.py --init --config 5 --steps 5 --warmup 3 >> gpurun_out/r03/bench_all.jsonl 2>> gpurun_out/r03/init.err
timeout 600 python bench.py --ingest --config 5 --steps 5 --warmup 3 >> gpurun_out/r03/bench_all.jsonl 2>> gpurun_out/r03/ingest.err
wc -l gpurun_out/r03/bench_all.jsonl
python - <<'PY'
import json
for l in open("gpurun_out/r03/bench_all.jsonl"):
    d = json.loads(l)
    r = d.get("roofline", {})
    print(d["metric"][:70], d["value"], d["unit"], "e2e", (d.get("e2e") or {}).get("value"),
          "frac", r.get("frac"), "cpu", (d.get("cpu_baseline") or {}).get("value"), "clk", d.get("clocks", {}).get("sm_mhz"))
PY
