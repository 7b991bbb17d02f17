#!/bin/bash
# same box: psi triples in the loop (SPUMA_OPT_LOOP_PSI_GROUP = 3) vs pairs, and vs the previous build
mkdir -p gpurun_out
export SPUMA_LIBRARY=$PWD/build/ab_tri.so
timeout 900 python -m pytest tests/test_gpu_persistent.py -q -x > gpurun_out/r02am_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02am_tests.log
for r in 1 2 3; do
  export SPUMA_LIBRARY=$PWD/build/ab_psipf2.so; unset SPUMA_AB_OPTS
  timeout 300 python scripts/persistent_ab.py 200 3 2 4 2>>gpurun_out/r02am.err | sed "s/^/prev r$r /" >> gpurun_out/r02am.txt
  export SPUMA_LIBRARY=$PWD/build/ab_tri.so; export SPUMA_AB_OPTS=16=3
  timeout 300 python scripts/persistent_ab.py 200 3 2 4 2>>gpurun_out/r02am.err | sed "s/^/tri3 r$r /" >> gpurun_out/r02am.txt
  export SPUMA_AB_OPTS=16=2
  timeout 300 python scripts/persistent_ab.py 200 3 2 4 2>>gpurun_out/r02am.err | sed "s/^/tri2 r$r /" >> gpurun_out/r02am.txt
done
