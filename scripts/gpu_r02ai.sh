#!/bin/bash
# same box: balanced last round of pair tiles vs whole tiles; parity of the balanced build
mkdir -p gpurun_out
export SPUMA_LIBRARY=$PWD/build/ab_bal.so
timeout 900 python -m pytest tests/test_gpu_persistent.py -q -x > gpurun_out/r02ai_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02ai_tests.log
for r in 1 2 3; do
for v in psipf2 bal; do
  export SPUMA_LIBRARY=$PWD/build/ab_$v.so
  timeout 300 python scripts/persistent_ab.py 200 3 2 4 2>>gpurun_out/r02ai.err | sed "s/^/$v r$r /" >> gpurun_out/r02ai.txt
done
done
