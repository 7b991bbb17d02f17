#!/bin/bash
# the loop below half residency: 318^3 lattice (26 % of rA on chip) and C4 64M ELL (13 %), loop vs graph
mkdir -p gpurun_out
export SPUMA_LIBRARY=$PWD/build/ab_res0.so
timeout 600 python scripts/l2_size_ab.py cube:318 3,2,4 0,2,0 3,2,0 2>&1 | sed "s/^/res0 /" >> gpurun_out/r02bh.txt
