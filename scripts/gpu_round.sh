#!/bin/bash
# One GPU-box pass: the GPU test suite, every bench leg, and the ncu captures
# summarised under profiles/ (outputs in gpurun_out/r02/).
set -x
mkdir -p gpurun_out/r02
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02/pytest_gpu.log 2>&1; tail -3 gpurun_out/r02/pytest_gpu.log
for c in 3 1 2 4 5; do timeout 900 python bench.py --config $c --steps 10 --warmup 3 >> gpurun_out/r02/bench.jsonl 2> gpurun_out/r02/bench_$c.err; done
timeout 600 python bench.py --oos --steps 10 --warmup 3 >> gpurun_out/r02/bench.jsonl 2>> gpurun_out/r02/bench_oos.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 >> gpurun_out/r02/bench.jsonl 2>> gpurun_out/r02/bench_ref.err
timeout 900 python bench.py --init --config 3 --steps 3 --warmup 3 --no-cpu-baseline >> gpurun_out/r02/bench.jsonl 2>> gpurun_out/r02/init.err
timeout 600 python bench.py --init --config 5 --steps 5 --warmup 3 >> gpurun_out/r02/bench.jsonl 2>> gpurun_out/r02/init.err
timeout 600 python bench.py --ingest --config 5 --steps 5 --warmup 3 >> gpurun_out/r02/bench.jsonl 2>> gpurun_out/r02/ingest.err
wc -l gpurun_out/r02/bench.jsonl
ncu --set full --clock-control none --import-source on -k regex:matvec_sym -c 1 -o gpurun_out/r02/init_matvec_cfg3 timeout 600 python scripts/time_init.py 3 > gpurun_out/r02/ncu_init.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"pack|combine" -c 20 --csv --log-file gpurun_out/r02/ingest_launches.csv timeout 600 python bench.py --ingest --config 5 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/r02/ncu_ingest.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02/launches_cfg3.csv timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02/ncu_launches3.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 50 --csv --log-file gpurun_out/r02/launches_cfg1.csv timeout 600 python bench.py --config 1 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02/ncu_launches1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:jofc_pass_kernel -s 3 -c 1 -o gpurun_out/r02/pass_kernel_cfg3 timeout 600 python scripts/diag_pass.py --config 3 --modes 0 --iters 5 > gpurun_out/r02/ncu_pass.log 2>&1
ls -la gpurun_out/r02
