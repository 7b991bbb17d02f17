#!/bin/bash
# final-code stability: the bench twice more, and C4 (64M perturbed + permuted, RCM) on one GPU
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/r02bd_gpu.txt 2>&1
for r in 1 2; do timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r02bd_bench_$r.json 2>> gpurun_out/r02bd.err; done
timeout 1500 python scripts/sweep.py C4 > gpurun_out/r02bd_c4.jsonl 2>> gpurun_out/r02bd.err
