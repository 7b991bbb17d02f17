#!/bin/bash
mkdir -p gpurun_out
for v in cur head; do
  if [ $v = cur ]; then unset SPUMA_LIBRARY; else export SPUMA_LIBRARY=$PWD/build/ab_$v.so; fi
  timeout 400 python scripts/l2_size_ab.py cube:252 3,2,4 2>&1 | sed "s/^/$v /" >> gpurun_out/r02ax.txt
  timeout 300 python scripts/persistent_ab.py 200 3 2 4 2>>gpurun_out/r02ax.err | sed "s/^/$v 200 /" >> gpurun_out/r02ax.txt
done
