#!/bin/bash
# OOS persistent solve: parity tests, bench --oos A/B against the per-update kernel (gpurun_out/oosp/).
mkdir -p gpurun_out/oosp
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_oos_c5.py tests/test_gpu_acceptance.py -k "oos or gate8" -x -q > gpurun_out/oosp/tests.log 2>&1; echo "rc=$?" >> gpurun_out/oosp/tests.log
tail -15 gpurun_out/oosp/tests.log
JOFC_OOSP_DEBUG=1 timeout 300 python bench.py --oos --steps 5 --warmup 3 --no-cpu-baseline 2>&1 >/dev/null | grep oosp | sort | uniq -c
for v in 4 3; do echo "v=$v $(JOFC_OOS_KERNEL=$v timeout 300 python bench.py --oos --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["e2e"]["value"])')"; done
for R in 512 256; do for G in 7 8 16; do
echo "G=$G R=$R $(JOFC_OOSP_G=$G JOFC_OOSP_ROWS=$R timeout 300 python bench.py --oos --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"])')"
done; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:oos_solve -c 1 -o gpurun_out/oosp/oosp python bench.py --oos --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/oosp/ncu.log 2>&1
tail -2 gpurun_out/oosp/ncu.log
