#!/bin/bash
# same box: update phase one vs two tiles ahead (both with the psi-pair prefetch)
mkdir -p gpurun_out
for r in 1 2 3; do
for v in psipf2 b2; do
  export SPUMA_LIBRARY=$PWD/build/ab_$v.so
  timeout 300 python scripts/persistent_ab.py 200 3 2 4 2>>gpurun_out/r02ah.err | sed "s/^/$v r$r /" >> gpurun_out/r02ah.txt
done
done
