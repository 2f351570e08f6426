#!/bin/bash
mkdir -p gpurun_out/oosp_diag
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_oos_c5.py tests/test_gpu_acceptance.py -k "oos or gate8" -x -q 2>&1 | tail -2
for R in 512 256 128; do for n in diag default; do
  lib=paper_1502_03391_b200/libjofc_gpu_$n.so; [ $n = default ] && lib=paper_1502_03391_b200/libjofc_gpu.so
  echo "$n R=$R $(JOFC_OOSP_ROWS=$R JOFC_GPU_LIB=$PWD/$lib timeout 300 python bench.py --oos --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["update_us"])')"
done; done | tee gpurun_out/oosp_diag/diag.txt
