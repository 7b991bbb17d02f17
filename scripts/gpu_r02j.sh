#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "amul or pcg_all" > gpurun_out/e16_tests.log 2>&1; tail -2 gpurun_out/e16_tests.log
timeout 900 python scripts/unstructured_ab.py 100 200 > gpurun_out/e16_ab.jsonl 2> gpurun_out/e16_ab.err; cat gpurun_out/e16_ab.jsonl
SPUMA_FULL_SIZE=1 timeout 2400 python -m pytest tests/test_gpu_full_size.py -q -s > gpurun_out/full_size_c4.log 2>&1; tail -14 gpurun_out/full_size_c4.log
