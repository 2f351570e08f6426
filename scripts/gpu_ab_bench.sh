#!/bin/bash
# Sustained (power-capped) A/B of builds on the C3 bench line, interleaved reps.
mkdir -p gpurun_out/ab_bench
for rep in 1 2 3; do for n in default ${VARIANTS}; do
  lib=paper_1502_03391_b200/libjofc_gpu_$n.so; [ $n = default ] && lib=paper_1502_03391_b200/libjofc_gpu.so
  echo "$n rep$rep $(JOFC_GPU_LIB=$PWD/$lib timeout 300 python bench.py --config ${CFG:-3} --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["avg_launch_ms"], d["clocks"]["sm_mhz"])')"
done; done | tee gpurun_out/ab_bench/ab.txt
