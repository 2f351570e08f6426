#!/bin/bash
# Round-5 (repo round 2) end sweep on one box: every bench leg, the reference arm,
# the C3 launch list and an ncu --set full capture of one identity-form C3 pass.
O=gpurun_out/r05
mkdir -p $O
: > $O/bench_all.jsonl
for c in 3 4 1 2 5; do timeout 900 python bench.py --config $c --steps 10 --warmup 3 >> $O/bench_all.jsonl 2> $O/bench_$c.err; done
timeout 600 python bench.py --oos --steps 10 --warmup 3 >> $O/bench_all.jsonl 2>> $O/bench_oos.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 >> $O/bench_all.jsonl 2>> $O/bench_ref.err
timeout 900 python bench.py --init --config 3 --steps 3 --warmup 3 --no-cpu-baseline >> $O/bench_all.jsonl 2>> $O/init.err
timeout 600 python bench.py --init --config 5 --steps 5 --warmup 3 >> $O/bench_all.jsonl 2>> $O/init.err
timeout 600 python bench.py --ingest --config 5 --steps 5 --warmup 3 >> $O/bench_all.jsonl 2>> $O/ingest.err
python - <<'PY'
import json
for l in open("gpurun_out/r05/bench_all.jsonl"):
    d = json.loads(l)
    r = d.get("roofline", {})
    print(d.get("impl", "ours"), d["metric"][:60], d["value"], d["unit"], "e2e", (d.get("e2e") or {}).get("value"),
          "frac", r.get("frac"), "cpu", (d.get("cpu_baseline") or {}).get("value"), "clk", d.get("clocks", {}).get("sm_mhz"))
PY
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_cfg3.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $O/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:jofc_pass_kernel -s 5 -c 1 -o $O/pass_cfg3 python scripts/diag_pass.py --config 3 --modes 0 --its 19 --iters 1 > $O/ncu_pass.log 2>&1
tail -2 $O/ncu_pass.log
