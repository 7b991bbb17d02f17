#!/bin/bash
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/r02y_gpu.txt 2>&1
timeout 300 python scripts/persistent_ab.py 200 0,3 2 4 > gpurun_out/r02y_200.jsonl 2>&1
timeout 600 python scripts/l2_size_ab.py cube:252 0,2,0 3,2,4 3,2,0 0,2,0 3,2,4 > gpurun_out/r02y_252.jsonl 2>&1
timeout 900 python -m pytest tests/test_gpu_persistent.py -q > gpurun_out/r02y_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02y_tests.log
timeout 900 python scripts/l2_size_ab.py C4 0,2,0 3,2,4 0,2,0 3,2,4 > gpurun_out/r02y_c4.jsonl 2>&1
