#!/bin/bash
# A/B of allocator flags: microbench timing, profile-build counters, apps
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); from paper_1810_11765_b200 import build; build.build(profile=True)" > gpurun_out/build.log 2>&1
rm -f gpurun_out/ab.log
for rep in 1 2 3; do for f in $1; do timeout -s KILL 120 python scripts/prof_mb.py $f 5 1 >> gpurun_out/ab.log 2>&1; done; done
for f in $1; do DSR_LIBPATH=paper_1810_11765_b200/_build/libdsr_prof.so timeout -s KILL 120 python scripts/prof_mb.py $((f | 4)) 5 1 >> gpurun_out/ab.log 2>&1; done
for f in $1; do timeout -s KILL 300 python scripts/ab_apps.py $f >> gpurun_out/ab.log 2>&1; done
