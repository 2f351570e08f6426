#!/bin/bash
# Sustained (power-capped) A/B of an experimental build against the shipped one:
# bench.py C3/C4 lines, interleaved.
for rep in 1 2; do
  for lib in libjofc_gpu.so libjofc_gpu_exp.so; do
    for c in "$@"; do
      echo -n "$lib cfg$c "
      JOFC_GPU_LIB=paper_1502_03391_b200/$lib timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e \
        | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['avg_launch_ms'], d['clocks']['sm_mhz'])"
    done
  done
done
