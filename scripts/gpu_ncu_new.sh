#!/bin/bash
mkdir -p gpurun_out
timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:k_mb_new -s 2 -c 1 -o gpurun_out/r01_mb_new_v2 -f python scripts/prof_targets.py mb > gpurun_out/ncu1.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu1.log
