#!/bin/bash
# Round-7 sweep (repo round 2, re-entry after the container was re-created): GPU suite, smoke,
# the default bench line, the reference arm, every other bench leg, and the C3 launch list,
# all on the libraries rebuilt from the committed sources.
O=gpurun_out/r07
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/gputest.log 2>&1; echo "gputest rc=$?" >> $O/gputest.log
tail -3 $O/gputest.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
python -c "import json; d=json.load(open('$O/bench.json')); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['clocks'])"
timeout 900 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
python -c "import json; d=json.load(open('$O/bench_ref.json')); print(d['value'], d['metric'], d.get('product_libraries_loaded'))"
rm -f $O/bench_other.jsonl
for c in 1 2 4 5; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline >> $O/bench_other.jsonl 2>> $O/bench_other.err; done
timeout 600 python bench.py --oos --steps 10 --warmup 3 >> $O/bench_other.jsonl 2>> $O/bench_other.err
python -c "
import json
for l in open('$O/bench_other.jsonl'):
    d=json.loads(l); print(d['metric'], d['value'], d['e2e']['value'], d['roofline'].get('frac'), d['clocks'].get('sm_mhz'), d['clocks'].get('power_w'))"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_cfg3.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $O/ncu_launch.log 2>&1
echo done
