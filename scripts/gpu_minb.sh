#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/prof_mb.log
for f in 0 128 384 0 128 384; do echo "== flags $f" >> gpurun_out/prof_mb.log; timeout -s KILL 60 python scripts/prof_mb.py $f 5 1 >> gpurun_out/prof_mb.log 2>&1; done
timeout -s KILL 60 python scripts/prof_mb.py 132 5 1 >> gpurun_out/prof_mb.log 2>&1
