#!/bin/bash
mkdir -p gpurun_out
free -g > gpurun_out/free.txt; nproc >> gpurun_out/free.txt; lscpu | grep "Model name" >> gpurun_out/free.txt
timeout 1800 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 1200 python scripts/sweep.py C1 C2 C5 > gpurun_out/sweep.jsonl 2> gpurun_out/sweep.err
echo done
