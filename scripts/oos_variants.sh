#!/bin/bash
# OOS pass-kernel variants (compile-time switches, `make exp`) timed by
# bench.py --oos; each variant twice, interleaved, on one box.
VARIANTS=("${@:-}")
[ ${#VARIANTS[@]} -eq 0 ] && VARIANTS=("")
for rep in 1 2; do
for v in "${VARIANTS[@]}"; do
  make -s exp EXP="$v" > /dev/null 2>&1 || { echo "build failed: $v"; continue; }
  echo -n "[$v] "
  JOFC_GPU_LIB=paper_1502_03391_b200/libjofc_gpu_exp.so timeout 300 python bench.py --oos --steps 20 --warmup 3 --no-cpu-baseline \
    | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['clocks']['sm_mhz'])"
done
done
