#!/bin/bash
# Pass-kernel time vs the band cost of the CTA range balancing (JOFC_BAND_COST).
for c in "$@"; do
  for bc in ${BC:-0 1 2 4 8}; do
    echo -n "band_cost=$bc "; JOFC_BAND_COST=$bc timeout 300 python scripts/diag_pass.py --config $c --modes 0 2>&1 | tail -1
  done
done
