#!/bin/bash
# windows over the first 83 MB of a vector larger than the persisting set-aside vs no window
mkdir -p gpurun_out
for v in final l2pre; do
  export SPUMA_LIBRARY=$PWD/build/ab_$v.so
  timeout 500 python scripts/l2_size_ab.py cube:318 0,2,0 0,1,0 2>&1 | sed "s/^/$v /" >> gpurun_out/r02bb.txt
  timeout 400 python scripts/l2_size_ab.py cube:252 3,2,4 3,2,1 2>&1 | sed "s/^/$v /" >> gpurun_out/r02bb.txt
done
