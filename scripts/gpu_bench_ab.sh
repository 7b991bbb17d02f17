#!/bin/bash
# same-box A/B of the bench step: Amul variant 8 vs 10, alternating sweeps on/off
mkdir -p gpurun_out
for r in 1 2; do
  for v in 8 10; do
    for a in 1 0; do
      timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --amul-variant $v --alt-sweep $a > gpurun_out/ab_v${v}_a${a}_r${r}.json 2>/dev/null
      python -c "import json,sys; d=json.load(open('gpurun_out/ab_v${v}_a${a}_r${r}.json')); print('round $r variant $v alt $a', round(d['value']/1e10,4), 'e10', d['config']['phase_avg_ms'], d['clocks']['sm_mhz'])"
    done
  done
done
