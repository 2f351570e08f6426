#!/bin/bash
mkdir -p gpurun_out/r05b
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r05b/gputest.log 2>&1; echo "gputest rc=$?" >> gpurun_out/r05b/gputest.log
tail -3 gpurun_out/r05b/gputest.log
timeout 300 python bench.py --oos --steps 10 --warmup 3 > gpurun_out/r05b/bench_oos.jsonl 2> gpurun_out/r05b/bench_oos.err
python -c "import json; d=json.load(open('gpurun_out/r05b/bench_oos.jsonl')); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['roofline']['kernel'], d.get('cpu_baseline',{}).get('value'))"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:oos_solve -c 1 -o gpurun_out/r05b/oosp python bench.py --oos --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/r05b/ncu.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r05b/oos_launches.csv python bench.py --oos --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
tail -3 gpurun_out/r05b/oos_launches.csv
