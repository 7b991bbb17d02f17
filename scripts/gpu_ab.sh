#!/bin/bash
mkdir -p gpurun_out
for i in 1 2; do
for L in libspuma libspuma_c974b1d libspuma_nopdl libspuma_nodual libspuma_neither; do
SPUMA_LIBRARY=$PWD/paper_2512_22215_b200/$L.so VARIANTS=8 timeout 300 python scripts/amul_variants.py 200 2>&1 | sed "s/^/$L /" >> gpurun_out/ab.log
done; done
echo done
