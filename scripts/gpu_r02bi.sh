#!/bin/bash
# same box (896-thread loop): the update two tiles ahead vs one
mkdir -p gpurun_out
for r in 1 2 3; do
for v in final b2x; do
  export SPUMA_LIBRARY=$PWD/build/ab_$v.so
  timeout 300 python scripts/persistent_ab.py 200 3 2 4 2>>gpurun_out/r02bi.err | sed "s/^/$v r$r /" >> gpurun_out/r02bi.txt
done
done
