#!/bin/bash
# A/B the current library against an older in-tree build on the same box
mkdir -p gpurun_out
for i in 1 2 3; do
VARIANTS=8 timeout 300 python scripts/amul_variants.py 200 >> gpurun_out/ab_new.log 2>&1
SPUMA_LIBRARY=$PWD/paper_2512_22215_b200/libspuma_c974b1d.so VARIANTS=8 timeout 300 python scripts/amul_variants.py 200 >> gpurun_out/ab_old.log 2>&1
done
echo done
