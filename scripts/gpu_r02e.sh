#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_lattice.py -q -x > gpurun_out/lattice_tests.log 2>&1; tail -1 gpurun_out/lattice_tests.log
for r in 1 2; do for v in 12 14; do timeout 300 python scripts/loop_overhead.py 200 0=$v 2>/dev/null | head -1 | cut -c1-200; done; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_amul_dot" -s 20 -c 2 -o gpurun_out/prof_v14 \
    python scripts/loop_overhead.py 200 0=14 > gpurun_out/ncu_v14.log 2>&1
echo done
