#!/bin/bash
mkdir -p gpurun_out
( while true; do free -g | awk 'NR==2{print $3}' >> gpurun_out/c4_mem.txt; sleep 10; done ) &
MP=$!
timeout 2400 python scripts/sweep.py C4 > gpurun_out/sweep_c4.jsonl 2> gpurun_out/sweep_c4.err
kill $MP
echo done
