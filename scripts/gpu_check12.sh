#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
rm -f gpurun_out/prof_mb.log
for a in "0 5 1" "16 5 1" "0 2 1" "16 2 1" "0 5 1"; do timeout -s KILL 60 python scripts/prof_mb.py $a >> gpurun_out/prof_mb.log 2>&1; done
timeout -s KILL 600 ncu --set full --import-source on --clock-control none -k regex:k_mb_new -s 2 -c 1 -o gpurun_out/r01_mb_new_res python scripts/prof_targets.py mb > gpurun_out/ncu1.log 2>&1
