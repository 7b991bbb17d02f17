#!/bin/bash
# same box: grid barrier arriving once per thread-block-cluster pair vs once per CTA
mkdir -p gpurun_out
export SPUMA_LIBRARY=$PWD/build/ab_cl2.so
timeout 900 python -m pytest tests/test_gpu_persistent.py -q -x > gpurun_out/r02be_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02be_tests.log
for r in 1 2 3; do
for v in final cl2; do
  export SPUMA_LIBRARY=$PWD/build/ab_$v.so
  for n in 30 200; do
    timeout 300 python scripts/persistent_ab.py $n 3 2 4 2>>gpurun_out/r02be.err | sed "s/^/$v r$r /" >> gpurun_out/r02be.txt
  done
done
done
