#!/bin/bash
# Fused-epilogue threshold experiment: it/s of the small configs with the
# epilogue fused into the pass kernel (n <= N) or separate (N = 0).
for c in 1 2 5; do
  for N in 0 100000; do
    echo -n "cfg$c fuse_n<=$N "
    JOFC_FUSE_EPI_N=$N timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['gpu_launches'])"
  done
done
