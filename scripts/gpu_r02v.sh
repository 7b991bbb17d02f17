#!/bin/bash
# same box: HEAD loop (base) vs pre-barrier prefetch (pf) vs prefetch + value-as-flag barrier (bar2)
mkdir -p gpurun_out
for r in 1 2 3; do
for v in base pf bar2; do
  if [ $v = base ]; then unset SPUMA_LIBRARY; else export SPUMA_LIBRARY=$PWD/build/ab_$v.so; fi
  timeout 300 python scripts/persistent_ab.py 200 3 2 4 2>>gpurun_out/r02v.err | sed "s/^/$v r$r /" >> gpurun_out/r02v.txt
done
done
export SPUMA_LIBRARY=$PWD/build/ab_bar2.so
timeout 600 python -m pytest tests/test_gpu_persistent.py -q -x > gpurun_out/r02v_bar2_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02v_bar2_tests.log
