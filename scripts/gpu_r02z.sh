#!/bin/bash
# grid-barrier polling A/B (same box): barrier-dominated small cubes and the bench cube
mkdir -p gpurun_out
for r in 1 2; do
for v in poll0 poll1 poll2; do
  export SPUMA_LIBRARY=$PWD/build/ab_$v.so
  for n in 30 100 200; do
    timeout 300 python scripts/persistent_ab.py $n 3 2 4 2>>gpurun_out/r02z.err | sed "s/^/$v r$r /" >> gpurun_out/r02z.txt
  done
done
done
