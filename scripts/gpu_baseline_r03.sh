#!/bin/bash
# Round-3 (repo round 2) first box call: baseline pass timings + sanitizer logs.
mkdir -p gpurun_out/r03
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/r03/smi.txt
for c in 3 4 5 2; do timeout 300 python scripts/diag_pass.py --config $c --modes 0 --iters 20 2>&1 | tail -1; done > gpurun_out/r03/diag_base.txt
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python scripts/sanitize.py > gpurun_out/r03/sanitize_$tool.log 2>&1
  echo "$tool exit $?" >> gpurun_out/r03/sanitize_summary.txt
done
cat gpurun_out/r03/diag_base.txt gpurun_out/r03/sanitize_summary.txt
