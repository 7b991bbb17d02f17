#!/bin/bash
mkdir -p gpurun_out
python scripts/l2_probe.py
for r in 1 2; do for v in 0 2 3 1; do echo "l2=$v $(timeout 300 python scripts/loop_overhead.py 200 8=$v 2>/dev/null | head -1 | cut -c1-200)"; done; done
