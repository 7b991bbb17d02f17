#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_persistent.py -q -x > gpurun_out/r02s_persistent.log 2>&1; echo "rc=$?" >> gpurun_out/r02s_persistent.log
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/r02s_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02s_pytest_gpu.log
