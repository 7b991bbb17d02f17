#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_robustness.py tests/test_gpu_gamg.py -q > gpurun_out/r02az_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02az_tests.log
timeout 600 python scripts/small_threshold_ab.py > gpurun_out/r02az_small.jsonl 2> gpurun_out/r02az.err
timeout 900 python scripts/sweep.py C1 > gpurun_out/r02az_c1.jsonl 2>> gpurun_out/r02az.err
