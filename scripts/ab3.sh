#!/bin/bash
# Interleaved timing of several builds: scripts/ab3.sh "LIB1 LIB2 ..." cfg...
LIBS=$1; shift
for rep in 1 2 3; do
  for lib in $LIBS; do
    for c in "$@"; do
      echo -n "$(basename $lib) "
      JOFC_GPU_LIB=$lib timeout 300 python scripts/diag_pass.py --config $c --modes 0 2>&1 | tail -1
    done
  done
done
