#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python scripts/amul_variants.py 200 > gpurun_out/variants.log 2>&1
timeout 600 python scripts/amul_variants.py 100 --permute --renumber > gpurun_out/variants_1M.log 2>&1
for v in ${PROFILE_VARIANTS:-5 7}; do
VARIANTS=$v timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_amul_dot -s 20 -c 1 -o gpurun_out/prof_v$v \
    python scripts/amul_variants.py 200 > gpurun_out/ncu_v$v.log 2>&1
done
echo done
