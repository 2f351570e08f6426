#!/bin/bash
# Interleaved pass-kernel timing of several libraries: scripts/ab3lib.sh "cfgs" lib...
CFGS=$1; shift
for rep in 1 2 3; do
  for lib in "$@"; do
    for c in $CFGS; do
      echo -n "$(basename $lib) "
      JOFC_GPU_LIB=$lib timeout 300 python scripts/diag_pass.py --config $c --modes 0 --its ${ITS:-0} 2>&1 | tail -1
    done
  done
done
