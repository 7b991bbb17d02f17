#!/bin/bash
mkdir -p gpurun_out
for r in 1 2; do
for v in bar1 t768; do
  export SPUMA_LIBRARY=$PWD/build/ab_$v.so
  timeout 300 python scripts/persistent_ab.py 200 3 0 0,3,4,1 2>>gpurun_out/r02r.err | sed "s/^/$v r$r /" >> gpurun_out/r02r.txt
done
done
unset SPUMA_LIBRARY
timeout 300 python scripts/persistent_ab.py 200 0 2 2>>gpurun_out/r02r.err | sed "s/^/graph_l2rA /" >> gpurun_out/r02r.txt
