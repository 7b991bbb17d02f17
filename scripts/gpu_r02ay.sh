#!/bin/bash
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/r02ay_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02ay_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02ay_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r02ay_smoke.log
timeout 600 python scripts/small_threshold_ab.py > gpurun_out/r02ay_small.jsonl 2> gpurun_out/r02ay.err
timeout 900 python scripts/sweep.py C1 > gpurun_out/r02ay_c1.jsonl 2>> gpurun_out/r02ay.err
timeout 600 python scripts/gamg_tail_ab.py > gpurun_out/r02ay_gamg_tail.jsonl 2>> gpurun_out/r02ay.err
