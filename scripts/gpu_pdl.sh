#!/bin/bash
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for i in 1 2; do
PDL=0 VARIANTS=8 timeout 300 python scripts/amul_variants.py 200 >> gpurun_out/pdl.log 2>&1
PDL=1 VARIANTS=8 timeout 300 python scripts/amul_variants.py 200 >> gpurun_out/pdl.log 2>&1
done
timeout 600 python scripts/sweep.py C1 > gpurun_out/sweep_c1.jsonl 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
echo done
