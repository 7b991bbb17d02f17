#!/bin/bash
# ncu --set full of the top kernels of the §8(f) solvers
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_gamg_post -s 19 -c 1 \
  -o gpurun_out/prof_gamg_post python scripts/gamg_profile.py 200 1 > gpurun_out/ncu_gamg_post.log 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_gamg_scale -s 19 -c 1 \
  -o gpurun_out/prof_gamg_scale python scripts/gamg_profile.py 200 1 > gpurun_out/ncu_gamg_scale.log 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_ilu_fwd -c 1 \
  -o gpurun_out/prof_ilu_fwd python scripts/precond_profile.py 100 > gpurun_out/ncu_ilu_fwd.log 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/precond_launches.csv python scripts/precond_profile.py 100 > gpurun_out/precond_prof.log 2>&1
ls -la gpurun_out/*.ncu-rep; tail -2 gpurun_out/ncu_gamg_post.log gpurun_out/ncu_ilu_fwd.log
