#!/bin/bash
mkdir -p gpurun_out
export SPUMA_LIBRARY=$PWD/build/ab_final.so
for r in 1 2 3; do
  timeout 600 python scripts/persistent_ab.py 200 3 2 4,1 2>>gpurun_out/r02bl.err | sed "s/^/r$r /" >> gpurun_out/r02bl.txt
done
timeout 600 python scripts/l2_size_ab.py cube:126 3,2,4 3,2,1 2>&1 | sed "s/^/126 /" >> gpurun_out/r02bl.txt
timeout 600 python scripts/l2_size_ab.py cube:159 3,2,4 3,2,1 2>&1 | sed "s/^/159 /" >> gpurun_out/r02bl.txt
