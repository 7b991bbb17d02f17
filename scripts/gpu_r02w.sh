#!/bin/bash
# persistent loop with ELL rows: tests, then the C1/C2/C5 and C4 sweeps, graph batches (0) vs loop (3)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/r02w_gpu.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_persistent.py -q > gpurun_out/r02w_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02w_tests.log
timeout 1500 python scripts/sweep.py C1 C2 C5 --modes=0,3 > gpurun_out/r02w_sweep.jsonl 2> gpurun_out/r02w_sweep.err
timeout 1500 python scripts/sweep.py C4 --modes=0,3 > gpurun_out/r02w_sweep_c4.jsonl 2> gpurun_out/r02w_sweep_c4.err
