#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_lattice.py -q -x > gpurun_out/inner_tests.log 2>&1; tail -1 gpurun_out/inner_tests.log
for r in 1 2 3; do
  unset SPUMA_LIBRARY; echo "inner   $(timeout 300 python scripts/loop_overhead.py 200 2>/dev/null | head -1 | cut -c1-230)"
  export SPUMA_LIBRARY=$PWD/build/ab_noinner.so; echo "noinner $(timeout 300 python scripts/loop_overhead.py 200 2>/dev/null | head -1 | cut -c1-230)"
done
