#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_lattice.py tests/test_gpu_gamg.py tests/test_gpu_gamg_multirank.py -q -x > gpurun_out/gamg_lat.log 2>&1; tail -2 gpurun_out/gamg_lat.log
for v in 12 10; do AMUL_VARIANT=$v timeout 900 python scripts/gamg_bench.py 200 2>&1 | cut -c1-420; done > gpurun_out/gamg_lat_ab.jsonl
cat gpurun_out/gamg_lat_ab.jsonl
