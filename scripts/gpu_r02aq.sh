#!/bin/bash
# another box: loop CTA size 896 vs 1024 (same-box, alternating, 4 rounds) + the bench once per build
mkdir -p gpurun_out
for r in 1 2 3 4; do
for v in h896 head; do
  export SPUMA_LIBRARY=$PWD/build/ab_$v.so
  timeout 300 python scripts/persistent_ab.py 200 3 2 4 2>>gpurun_out/r02aq.err | sed "s/^/$v r$r /" >> gpurun_out/r02aq.txt
done
done
for v in h896 head; do
  export SPUMA_LIBRARY=$PWD/build/ab_$v.so
  timeout 600 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/r02aq_bench_$v.json 2>>gpurun_out/r02aq.err
done
