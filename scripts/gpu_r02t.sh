#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_persistent.py tests/test_gpu_parity.py -q > gpurun_out/r02t_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02t_tests.log
for r in 1 2; do
for v in base disc; do
  if [ $v = base ]; then unset SPUMA_LIBRARY; else export SPUMA_LIBRARY=$PWD/build/ab_$v.so; fi
  timeout 300 python scripts/persistent_ab.py 200 3 2 4,0 2>>gpurun_out/r02t.err | sed "s/^/$v r$r /" >> gpurun_out/r02t.txt
done
done
unset SPUMA_LIBRARY
timeout 600 python bench.py > gpurun_out/r02t_bench.json 2> gpurun_out/r02t_bench.err
