#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_persistent.py tests/test_gpu_lattice.py tests/test_gpu_parity.py -q > gpurun_out/r02bm_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02bm_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02bm_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r02bm_smoke.log
timeout 900 python bench.py > gpurun_out/r02bm_bench.json 2> gpurun_out/r02bm_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02bm_bench_ref.json 2> gpurun_out/r02bm_bench_ref.err
