#!/bin/bash
# same box: loop CTA size 1024 (64 registers) vs 896 (72) vs 768 (80), with the psi-pair prefetch
mkdir -p gpurun_out
export SPUMA_LIBRARY=$PWD/build/ab_t896.so
timeout 900 python -m pytest tests/test_gpu_persistent.py -q -x > gpurun_out/r02an_tests896.log 2>&1; echo "rc=$?" >> gpurun_out/r02an_tests896.log
for r in 1 2 3; do
for v in head t896 t768b; do
  export SPUMA_LIBRARY=$PWD/build/ab_$v.so
  timeout 300 python scripts/persistent_ab.py 200 3 2 4 2>>gpurun_out/r02an.err | sed "s/^/$v r$r /" >> gpurun_out/r02an.txt
done
done
