#!/bin/bash
# allocator counters (DSR_F_STATS) for the microbench step, with/without reserve, r=5/2,
# from the profiling build (-DDSR_PROFILE, _build/libdsr_prof.so)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); from paper_1810_11765_b200 import build; build.build(profile=True)" > gpurun_out/build.log 2>&1
rm -f gpurun_out/prof_mb.log
export DSR_LIBPATH=$PWD/paper_1810_11765_b200/_build/libdsr_prof.so
for a in "4 5 1" "4 5 0" "4 2 1" "20 5 1" "0 5 1"; do timeout -s KILL 60 python scripts/prof_mb.py $a >> gpurun_out/prof_mb.log 2>&1; done
