#!/bin/bash
# OOS v2 pass variants: builds x waves (JOFC_OOS_KERNEL=2)
run() { echo -n "$1 waves=$2: "; JOFC_GPU_LIB=$1 JOFC_OOS_KERNEL=2 JOFC_OOS2_WAVES=$2 timeout 300 python bench.py --oos --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['update_us'])"; }
for lib in paper_1502_03391_b200/libjofc_gpu.so paper_1502_03391_b200/libjofc_gpu_o2_32_4.so paper_1502_03391_b200/libjofc_gpu_o2_32_6.so paper_1502_03391_b200/libjofc_gpu_o2_128_3.so; do
  for w in 1 2 4; do run $lib $w; done
done
echo -n "fused default: "; timeout 300 python bench.py --oos --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['update_us'])"
