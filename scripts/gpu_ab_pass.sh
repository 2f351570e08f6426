#!/bin/bash
# A/B of pass-kernel builds (libjofc_gpu_<name>.so) on C3/C4 identity-form passes, interleaved reps.
mkdir -p gpurun_out/ab_pass
for rep in 1 2 3; do for n in default ${VARIANTS}; do
  lib=paper_1502_03391_b200/libjofc_gpu_$n.so; [ $n = default ] && lib=paper_1502_03391_b200/libjofc_gpu.so
  for cfg in 3 4; do
    echo "$n rep$rep $(JOFC_GPU_LIB=$PWD/$lib timeout 300 python scripts/diag_pass.py --config $cfg --modes 0 --its 19 2>&1 | tail -1)"
  done
done; done | tee gpurun_out/ab_pass/ab.txt
