#!/bin/bash
# same box: lattice rows of the loop's Amul phase, pipelined (next chunk's streams ahead) vs not
mkdir -p gpurun_out
for r in 1 2 3; do
for v in latbase latpipe rdinl; do
  export SPUMA_LIBRARY=$PWD/build/ab_$v.so
  timeout 300 python scripts/persistent_ab.py 200 3 2 4 2>>gpurun_out/r02ad.err | sed "s/^/$v r$r /" >> gpurun_out/r02ad.txt
done
done
