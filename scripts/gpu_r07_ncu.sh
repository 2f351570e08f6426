#!/bin/bash
# Round-7 ncu --set full captures of the rebuilt libraries (each after its command ran clean
# without ncu in scripts/gpu_r07.sh): `pass` = one identity-form C3 pass and one C4 pass,
# `oos` = one C5 out-of-sample batch solve (two calls: the reports together exceed gpurun's
# 64 MiB return limit).
O=gpurun_out/r07
mkdir -p $O
if [ "$1" = pass ]; then
for c in 3 4; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:jofc_pass_kernel -s 5 -c 1 -o $O/pass_cfg$c python scripts/diag_pass.py --config $c --modes 0 --its 19 --iters 1 > $O/ncu_pass$c.log 2>&1; tail -1 $O/ncu_pass$c.log
done
else
timeout 600 ncu --set full --clock-control none --import-source on -k regex:oos_solve -c 1 -o $O/oosp python bench.py --oos --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu_oos.log 2>&1; tail -1 $O/ncu_oos.log
fi
ls -la $O/*.ncu-rep
