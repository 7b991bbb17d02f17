#!/bin/bash
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/sweep_gpu.txt 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench2.json 2> gpurun_out/bench2.err
timeout 1500 python scripts/sweep.py C1 C2 C5 > gpurun_out/sweep.jsonl 2> gpurun_out/sweep.err
timeout 1500 python scripts/sweep.py C4 > gpurun_out/sweep_c4.jsonl 2> gpurun_out/sweep_c4.err
cut -c1-200 gpurun_out/sweep.jsonl gpurun_out/sweep_c4.jsonl; cut -c1-300 gpurun_out/bench2.json
