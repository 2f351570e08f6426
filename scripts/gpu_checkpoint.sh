#!/bin/bash
# Checkpoint on one box: A/B of the pass kernel against the last baseline
# build, the GPU test suite, the default bench line, the reference arm.
mkdir -p gpurun_out/r03
bash scripts/ab3.sh "paper_1502_03391_b200/libjofc_gpu_base.so paper_1502_03391_b200/libjofc_gpu.so" 3 4 > gpurun_out/r03/ab_ckpt.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r03/pytest_ckpt.log 2>&1; tail -3 gpurun_out/r03/pytest_ckpt.log
timeout 900 python bench.py > gpurun_out/r03/bench_c3.jsonl 2> gpurun_out/r03/bench_c3.err; tail -c 3000 gpurun_out/r03/bench_c3.jsonl
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r03/bench_ref.jsonl 2> gpurun_out/r03/bench_ref.err; cat gpurun_out/r03/bench_ref.jsonl
cat gpurun_out/r03/ab_ckpt.txt
