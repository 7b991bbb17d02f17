#!/bin/bash
# ELL meshes: graph batches vs the persistent loop (C2 1M permuted + RCM, 8M perturbed permuted + RCM)
mkdir -p gpurun_out
timeout 900 python scripts/sweep.py C2 --modes=0,3 > gpurun_out/r02aa_c2.jsonl 2> gpurun_out/r02aa_c2.err
timeout 900 python scripts/l2_size_ab.py perm:200 0,2,0 3,2,4 3,2,0 0,2,0 3,2,4 > gpurun_out/r02aa_perm200.jsonl 2>&1
export SPUMA_LIBRARY=$PWD/build/ab_ellpipe.so
timeout 900 python scripts/l2_size_ab.py perm:200 3,2,4 > gpurun_out/r02aa_perm200_pipe.jsonl 2>&1
