#!/bin/bash
# 252^3 (half of rA on chip): which change slowed the loop there?
mkdir -p gpurun_out
for v in latbase psipf2 head h896 cur; do
  if [ $v = cur ]; then unset SPUMA_LIBRARY; else export SPUMA_LIBRARY=$PWD/build/ab_$v.so; fi
  timeout 400 python scripts/l2_size_ab.py cube:252 3,2,4 0,2,0 2>&1 | sed "s/^/$v /" >> gpurun_out/r02av.txt
done
