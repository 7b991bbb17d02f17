#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gamg.py -q -x > gpurun_out/gamg_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gamg_pytest.log
tail -3 gpurun_out/gamg_pytest.log
for T in 0 1024 4096 16384; do
  GAMG_TAIL=$T python scripts/gamg_bench.py 100 128 200 2>&1 | grep -v two-stage | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['case'], 'cycles', d['gamg_cycles'], 'ms/cycle %.3f' % d['gamg_ms_per_cycle'], 'gamg_s %.4f' % d['gamg_solve_s'])"
done
