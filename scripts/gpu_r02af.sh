#!/bin/bash
# same box: TMA bulk L2 prefetch in the loop's lattice Amul phase, distance 1/2/4 CTA steps vs none
mkdir -p gpurun_out
python scripts/build_ab.py base0 > /dev/null 2>&1 || true
for r in 1 2; do
for v in latbase bpf1 bpf2 bpf4; do
  export SPUMA_LIBRARY=$PWD/build/ab_$v.so
  timeout 300 python scripts/persistent_ab.py 200 3 2 4 2>>gpurun_out/r02af.err | sed "s/^/$v r$r /" >> gpurun_out/r02af.txt
done
done
