#!/bin/bash
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/r02bj_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02bj_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02bj_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r02bj_smoke.log
timeout 900 python bench.py > gpurun_out/r02bj_bench.json 2> gpurun_out/r02bj_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02bj_launches.csv \
    python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/r02bj_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_pcg_loop" -c 1 -o gpurun_out/r02bj_prof_loop \
    python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/r02bj_ncu_full.log 2>&1
timeout 1500 python scripts/sweep.py C1 C2 C5 > gpurun_out/r02bj_sweep.jsonl 2> gpurun_out/r02bj_sweep.err
