#!/bin/bash
# full GPU suite + smoke with the loop as default; C1/C5 sweep graph vs loop
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/r02ab_gpu.txt 2>&1
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/r02ab_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02ab_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02ab_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r02ab_smoke.log
timeout 1500 python scripts/sweep.py C1 C5 --modes=0,3 > gpurun_out/r02ab_sweep.jsonl 2> gpurun_out/r02ab_sweep.err
