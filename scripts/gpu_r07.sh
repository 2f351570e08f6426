#!/bin/bash
# Round-7 check (repo round 2, re-entry after the container was re-created): GPU suite, smoke,
# the default bench line and the reference arm on the rebuilt libraries.
O=gpurun_out/r07
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/gputest.log 2>&1; echo "gputest rc=$?" >> $O/gputest.log
tail -3 $O/gputest.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
python -c "import json; d=json.load(open('$O/bench.json')); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['clocks'])"
timeout 900 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
python -c "import json; d=json.load(open('$O/bench_ref.json')); print(d['value'], d['metric'], d.get('product_libraries_loaded'))"
echo done
