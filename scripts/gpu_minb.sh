#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/prof_mb.log
for a in "4 5 1" "4 5 0" "0 5 1"; do timeout -s KILL 60 python scripts/prof_mb.py $a >> gpurun_out/prof_mb.log 2>&1; done
