#!/bin/bash
# pass-kernel time of one build in diag modes (0 full, 3 no column reduction, 4 stream only)
LIB=${1:-paper_1502_03391_b200/libjofc_gpu.so}; shift
for c in "$@"; do
  JOFC_GPU_LIB=$LIB timeout 600 python scripts/diag_pass.py --config $c --modes 0,3,4 2>&1 | grep cfg
done
