#!/bin/bash
# same box: psi-pair loads prefetched one tile ahead in the loop's direction phase vs not
mkdir -p gpurun_out
for r in 1 2 3; do
for v in latbase psipf; do
  export SPUMA_LIBRARY=$PWD/build/ab_$v.so
  timeout 300 python scripts/persistent_ab.py 200 3 2 4 2>>gpurun_out/r02ag.err | sed "s/^/$v r$r /" >> gpurun_out/r02ag.txt
done
done
