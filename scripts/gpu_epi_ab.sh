#!/bin/bash
# 256- vs 1024-thread identity-form epilogue: parity subset, whole-solve A/B, epilogue launch times.
mkdir -p gpurun_out/epi
timeout 900 python -m pytest tests/test_gpu_fidelity_form.py tests/test_gpu_nccl.py tests/test_layout_shards.py tests/test_gpu_fuzz.py -x -q 2>&1 | tail -2
for rep in 1 2 3; do for v in 1 0; do for c in 4; do echo "small=$v rep$rep $(JOFC_WIDE_SMALL=$v python scripts/route_probe.py $c)"; done; done; done
for v in 1 0; do JOFC_WIDE_SMALL=$v ncu --metrics gpu__time_duration.sum -k regex:epilogue_wide -c 20 python scripts/route_probe.py 3 2>/dev/null | grep -E "duration" | awk -v v=$v '{s+=$3; n++} END {print "small=" v " epilogue avg us", s/n}'; done
