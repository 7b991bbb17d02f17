#!/bin/bash
# same box: two lattice rows per lane in the loop's Amul phase vs one
mkdir -p gpurun_out
export SPUMA_LIBRARY=$PWD/build/ab_r2.so
timeout 900 python -m pytest tests/test_gpu_persistent.py -q -x > gpurun_out/r02bg_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02bg_tests.log
for r in 1 2 3; do
for v in final r2; do
  export SPUMA_LIBRARY=$PWD/build/ab_$v.so
  timeout 300 python scripts/persistent_ab.py 200 3 2 4 2>>gpurun_out/r02bg.err | sed "s/^/$v r$r /" >> gpurun_out/r02bg.txt
done
done
