#!/bin/bash
# round 2 baseline: loop overhead probe, bench, PDL off A/B
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total,power.limit --format=csv > gpurun_out/gpu.txt 2>&1
timeout 600 python scripts/loop_overhead.py 200 > gpurun_out/loop_overhead.jsonl 2> gpurun_out/loop_overhead.err
timeout 600 python scripts/loop_overhead.py 200 2=0 >> gpurun_out/loop_overhead.jsonl 2>> gpurun_out/loop_overhead.err
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
cat gpurun_out/loop_overhead.jsonl; cut -c1-400 gpurun_out/bench.json
