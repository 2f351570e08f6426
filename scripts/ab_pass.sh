#!/bin/bash
# Interleaved A/B of pass-kernel time: scripts/ab_pass.sh LIB_A LIB_B cfg... (JOFC_GPU_LIB)
A=$1; B=$2; shift 2
for rep in 1 2 3; do
  for lib in $A $B; do
    for c in "$@"; do
      echo -n "$(basename $lib) "
      JOFC_GPU_LIB=$lib timeout 300 python scripts/diag_pass.py --config $c --modes 0 2>&1 | tail -1
    done
  done
done
