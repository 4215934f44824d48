#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/prof_mb.log
for a in "0 5 1 0" "0 5 1 0.02" "0 5 1 0.05" "0 5 1 0.1" "0 5 1 0.25" "0 2 1 0.05" "0 5 1 0"; do timeout -s KILL 60 python scripts/prof_mb.py $a >> gpurun_out/prof_mb.log 2>&1; done
timeout -s KILL 600 python -m pytest tests/test_gpu_allocator.py -x -q >> gpurun_out/prof_mb.log 2>&1
