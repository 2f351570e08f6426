#!/bin/bash
# OOS pass-kernel variants (compile-time switches) timed by bench.py --oos, A/B
# on one box: each variant twice, interleaved.
for rep in 1 2; do
for v in "-DJOFC_OOS_UNROLL=1" "-DJOFC_OOS_UNROLL=2" "-DJOFC_OOS_UNROLL=4" "-DJOFC_OOS_UNROLL=8"; do
  make -s exp EXP="$v" > /dev/null 2>&1 || { echo "build failed: $v"; continue; }
  echo -n "[$v] "
  JOFC_GPU_LIB=paper_1502_03391_b200/libjofc_gpu_exp.so timeout 300 python bench.py --oos --steps 20 --warmup 3 --no-cpu-baseline --no-e2e \
    | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['clocks']['sm_mhz'])"
done
done
