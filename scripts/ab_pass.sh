#!/bin/bash
# A/B of the pass kernel variants on one box: default vs JOFC_PASS_MMA=1.
for rep in 1 2; do
  for c in "$@"; do
    echo -n "vector  "; JOFC_PASS_MMA=0 timeout 300 python scripts/diag_pass.py --config $c --modes 0 2>&1 | tail -1
    echo -n "mma     "; JOFC_PASS_MMA=1 timeout 300 python scripts/diag_pass.py --config $c --modes 0 2>&1 | tail -1
  done
done
