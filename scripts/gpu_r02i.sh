#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_lattice.py -q -x -k fused > gpurun_out/fused_tests.log 2>&1; tail -2 gpurun_out/fused_tests.log
for r in 1 2; do for f in 0 3; do timeout 300 python scripts/loop_overhead.py 200 5=$f 2>/dev/null | head -1 | cut -c1-330; done; done
