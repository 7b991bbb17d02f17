#!/bin/bash
mkdir -p gpurun_out
for r in 1 2; do
for v in base bar1 xcg bar1xcg; do
  if [ $v = base ]; then unset SPUMA_LIBRARY; else export SPUMA_LIBRARY=$PWD/build/ab_$v.so; fi
  timeout 300 python scripts/persistent_ab.py 200 3 0 2>>gpurun_out/r02q.err | sed "s/^/$v r$r /" >> gpurun_out/r02q.txt
done
done
unset SPUMA_LIBRARY
timeout 300 python scripts/persistent_ab.py 200 0 2 2>>gpurun_out/r02q.err | sed "s/^/graph_l2rA /" >> gpurun_out/r02q.txt
