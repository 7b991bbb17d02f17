#!/bin/bash
# same box: the direction phase two tiles ahead (psi loads in place) vs one ahead (psi loads prefetched)
mkdir -p gpurun_out
export SPUMA_LIBRARY=$PWD/build/ab_c2.so
timeout 900 python -m pytest tests/test_gpu_persistent.py -q -x > gpurun_out/r02bc_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02bc_tests.log
for r in 1 2 3; do
for v in final c2; do
  export SPUMA_LIBRARY=$PWD/build/ab_$v.so
  timeout 300 python scripts/persistent_ab.py 200 3 2 4 2>>gpurun_out/r02bc.err | sed "s/^/$v r$r /" >> gpurun_out/r02bc.txt
done
done
