#!/bin/bash
# final code: the loop's L2 window target wA (default) vs pA vs rD vs none
mkdir -p gpurun_out
export SPUMA_LIBRARY=$PWD/build/ab_final.so
for r in 1 2; do
  timeout 600 python scripts/persistent_ab.py 200 3 2 4,1,3,0 2>>gpurun_out/r02bk.err | sed "s/^/r$r /" >> gpurun_out/r02bk.txt
done
