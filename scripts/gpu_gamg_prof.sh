#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/gamg_launches.csv python scripts/gamg_profile.py 200 3 > gpurun_out/gamg_prof.log 2>&1
echo "rc=$?" >> gpurun_out/gamg_prof.log
tail -3 gpurun_out/gamg_prof.log
