#!/bin/bash
# Short (full-clock) A/B of libjofc_gpu_exp.so (make exp EXP=...) against the
# shipped library: pass-kernel time from scripts/diag_pass.py, interleaved.
for rep in 1 2 3; do
  for lib in libjofc_gpu.so libjofc_gpu_exp.so; do
    for c in "$@"; do
      echo -n "$lib "
      JOFC_GPU_LIB=paper_1502_03391_b200/$lib timeout 300 python scripts/diag_pass.py --config $c --modes 0 2>&1 | tail -1
    done
  done
done
