#!/bin/bash
# persistent PCG loop: first run (A/B vs graph batches, lattice parity tests)
mkdir -p gpurun_out
timeout 300 python scripts/persistent_ab.py 100 0,1,2,3 2 > gpurun_out/r02o_ab100.jsonl 2> gpurun_out/r02o_ab100.err
timeout 300 python scripts/persistent_ab.py 200 0,1,2,3 2,0,1 > gpurun_out/r02o_ab200.jsonl 2> gpurun_out/r02o_ab200.err
timeout 600 python -m pytest tests/test_gpu_lattice.py -x -q > gpurun_out/r02o_lattice.log 2>&1
