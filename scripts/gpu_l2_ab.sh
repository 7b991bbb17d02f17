#!/bin/bash
# same-box A/B: deferred psi x L2 persisting window over pA
mkdir -p gpurun_out
python -c "import torch; p=torch.cuda.get_device_properties(0); print('L2', p.L2_cache_size)" 
for r in 1 2; do
  for cfg in "1 0" "0 0" "0 1" "1 1"; do
    set -- $cfg
    timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --defer-psi $1 --l2-persist $2 > gpurun_out/l2_d$1_p$2_r$r.json 2>gpurun_out/l2.err
    python -c "import json; d=json.load(open('gpurun_out/l2_d$1_p$2_r$r.json')); print('round $r defer $1 persist $2', round(d['value']/1e10,4), 'e10', {k: round(v*1e3,1) for k,v in d['config']['phase_avg_ms'].items()}, d['clocks']['sm_mhz'])"
  done
done
