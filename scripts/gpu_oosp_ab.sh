#!/bin/bash
# A/B of persistent-OOS variants (libjofc_gpu_<name>.so builds), 2 interleaved reps.
mkdir -p gpurun_out/oosp_ab
for rep in 1 2; do for n in default ${VARIANTS:-u2 c12u2 c8q4 q1u2 c12q4}; do
  lib=paper_1502_03391_b200/libjofc_gpu_$n.so; [ $n = default ] && lib=paper_1502_03391_b200/libjofc_gpu.so
  echo "$n rep$rep $(JOFC_GPU_LIB=$PWD/$lib JOFC_OOSP_DEBUG=1 timeout 300 python bench.py --oos --steps 10 --warmup 3 --no-cpu-baseline 2>gpurun_out/oosp_ab/$n.err | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"])') $(grep -m1 oosp gpurun_out/oosp_ab/$n.err | cut -c30-)"
done; done | tee gpurun_out/oosp_ab/ab.txt
