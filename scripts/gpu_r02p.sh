#!/bin/bash
mkdir -p gpurun_out
timeout 300 python scripts/persistent_ab.py 200 0,1,2,3 0 > gpurun_out/r02p_ab200.jsonl 2> gpurun_out/r02p_ab200.err
timeout 300 python scripts/persistent_ab.py 200 0 2 >> gpurun_out/r02p_ab200.jsonl 2>> gpurun_out/r02p_ab200.err
