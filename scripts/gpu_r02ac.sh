#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_persistent.py -q > gpurun_out/r02ac_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02ac_tests.log
timeout 900 python scripts/sweep.py C2 --modes=0,3 > gpurun_out/r02ac_c2.jsonl 2> gpurun_out/r02ac_c2.err
