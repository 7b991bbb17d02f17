#!/bin/bash
# ncu of the persistent loop: launch list (time per launch) + one --set full capture of k_pcg_loop
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02u_launches.csv \
    python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/r02u_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_pcg_loop" -c 1 -o gpurun_out/r02u_prof_loop \
    python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/r02u_ncu_full.log 2>&1
echo done
