#!/bin/bash
# same box (896-thread loop): psi triples vs pairs
mkdir -p gpurun_out
export SPUMA_LIBRARY=$PWD/build/ab_tri896.so
timeout 900 python -m pytest tests/test_gpu_persistent.py -q -x > gpurun_out/r02ao_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02ao_tests.log
for r in 1 2 3; do
  export SPUMA_LIBRARY=$PWD/build/ab_h896.so; unset SPUMA_AB_OPTS
  timeout 300 python scripts/persistent_ab.py 200 3 2 4 2>>gpurun_out/r02ao.err | sed "s/^/h896 r$r /" >> gpurun_out/r02ao.txt
  export SPUMA_LIBRARY=$PWD/build/ab_tri896.so; export SPUMA_AB_OPTS=16=3
  timeout 300 python scripts/persistent_ab.py 200 3 2 4 2>>gpurun_out/r02ao.err | sed "s/^/tri3 r$r /" >> gpurun_out/r02ao.txt
  export SPUMA_AB_OPTS=16=2
  timeout 300 python scripts/persistent_ab.py 200 3 2 4 2>>gpurun_out/r02ao.err | sed "s/^/tri2 r$r /" >> gpurun_out/r02ao.txt
done
