#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "deferred or pcg" > gpurun_out/defer_tests.log 2>&1; tail -1 gpurun_out/defer_tests.log
for r in 1 2; do for d in 1 2; do timeout 300 python scripts/loop_overhead.py 200 3=$d 2>/dev/null | head -1 | cut -c1-300; done; done
echo done
