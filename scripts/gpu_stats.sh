#!/bin/bash
# allocator counters (DSR_F_STATS) for the microbench step, with/without reserve, r=5/2
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
rm -f gpurun_out/prof_mb.log
for a in "4 5 1" "4 5 0" "4 2 1" "20 5 1" "0 5 1"; do timeout -s KILL 60 python scripts/prof_mb.py $a >> gpurun_out/prof_mb.log 2>&1; done
