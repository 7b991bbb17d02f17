#!/bin/bash
# round 2: lattice Amul parity + robustness + A/B of the hot-loop variants
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_robustness.py tests/test_gpu_lattice.py -q -x > gpurun_out/lattice_tests.log 2>&1; echo "rc=$?" >> gpurun_out/lattice_tests.log
tail -3 gpurun_out/lattice_tests.log
for v in 12 13 10; do timeout 300 python scripts/loop_overhead.py 200 0=$v 2>&1 | head -1; done > gpurun_out/variant_ab.jsonl
cat gpurun_out/variant_ab.jsonl
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/parity.log 2>&1; echo "rc=$?" >> gpurun_out/parity.log
tail -3 gpurun_out/parity.log
