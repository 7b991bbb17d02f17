#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_robustness.py tests/test_gpu_parity.py tests/test_gpu_gamg.py -q -x -k "small or shared or tail or gamg" > gpurun_out/small_tests.log 2>&1; tail -2 gpurun_out/small_tests.log
timeout 600 python scripts/sweep.py C1 > gpurun_out/c1.jsonl 2>&1; cut -c1-200 gpurun_out/c1.jsonl
