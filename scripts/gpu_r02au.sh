#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_persistent.py tests/test_gpu_lattice.py -q > gpurun_out/r02au_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02au_tests.log
timeout 600 python scripts/loop_grid_ab.py > gpurun_out/r02au_grid.jsonl 2> gpurun_out/r02au.err
timeout 600 python scripts/small_threshold_ab.py > gpurun_out/r02au_small.jsonl 2>> gpurun_out/r02au.err
