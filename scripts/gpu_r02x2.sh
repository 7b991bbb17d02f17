#!/bin/bash
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/r02x2_gpu.txt 2>&1
timeout 600 python scripts/l2_size_ab.py cube:252 0,0,0 0,2,0 3,2,0 3,2,4 3,0,4 3,0,1 > gpurun_out/r02x2_252.jsonl 2>&1
timeout 900 python scripts/l2_size_ab.py C4 0,0,0 0,2,0 3,0,0 3,0,4 > gpurun_out/r02x2_c4.jsonl 2>&1
for v in pfa1 pfa2 pfa3; do
  export SPUMA_LIBRARY=$PWD/build/ab_$v.so
  timeout 300 python scripts/persistent_ab.py 200 3 2 4 2>>gpurun_out/r02x2.err | sed "s/^/$v /" >> gpurun_out/r02x2_pfa.txt
done
unset SPUMA_LIBRARY
timeout 300 python scripts/persistent_ab.py 200 3 2 4 2>>gpurun_out/r02x2.err | sed "s/^/base /" >> gpurun_out/r02x2_pfa.txt
export SPUMA_LIBRARY=$PWD/build/ab_pfa2.so
timeout 300 python scripts/persistent_ab.py 200 3 2 4 2>>gpurun_out/r02x2.err | sed "s/^/pfa2 /" >> gpurun_out/r02x2_pfa.txt
