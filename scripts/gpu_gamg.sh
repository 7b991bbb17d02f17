#!/bin/bash
# GAMG parity + time to solution (+ optional launch list) on the GPU box
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/gamg_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_gamg.py -x -q > gpurun_out/gamg_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gamg_pytest.log
timeout 600 python scripts/gamg_bench.py ${GAMG_SIZES:-100 200} > gpurun_out/gamg_bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/gamg_bench.log
if [ -n "$GAMG_PROF" ]; then
  timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/gamg_launches.csv python scripts/gamg_profile.py 200 3 > gpurun_out/gamg_prof.log 2>&1
fi
tail -3 gpurun_out/gamg_pytest.log; python - <<'PY'
import json
for l in open('gpurun_out/gamg_bench.log'):
    if l.startswith('{'):
        d = json.loads(l); print(d['case'], 'cycles', d['gamg_cycles'], 'ms/cycle %.3f' % d['gamg_ms_per_cycle'],
              'gamg_s %.4f' % d['gamg_solve_s'], 'pcg_s %.4f' % d['pcg_solve_s'], 'pcg_it', d['pcg_iterations'])
    else:
        print(l.rstrip()[:300])
PY
