#!/bin/bash
# Interleaved A/B of whole bench lines (device it/s) for two builds:
# scripts/ab_bench.sh LIB_A LIB_B cfg...
A=$1; B=$2; shift 2
for rep in 1 2 3; do
  for lib in $A $B; do
    for c in "$@"; do
      echo -n "$(basename $lib) cfg$c "
      JOFC_GPU_LIB=$lib timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline'].get('iteration_ms'))"
    done
  done
done
