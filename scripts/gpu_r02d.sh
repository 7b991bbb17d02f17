#!/bin/bash
# round 2: lattice Amul A/B (occupancy, cache hints) + ncu of the hot-loop kernels
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_lattice.py -q -x > gpurun_out/lattice_tests.log 2>&1; tail -1 gpurun_out/lattice_tests.log
for r in 1 2; do
for lib in default ab_ctas5 ab_ctas3 ab_hint1 ab_hint2; do
  if [ $lib = default ]; then unset SPUMA_LIBRARY; else export SPUMA_LIBRARY=$PWD/build/$lib.so; fi
  echo "{\"lib\": \"$lib\", \"round\": $r, \"r\": $(timeout 300 python scripts/loop_overhead.py 200 2>/dev/null | head -1)}"
done; done > gpurun_out/lat_ab.jsonl
unset SPUMA_LIBRARY
cut -c1-250 gpurun_out/lat_ab.jsonl
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_amul_dot|k_direction|k_update" -s 60 -c 6 -o gpurun_out/prof_hot \
    python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
echo done
