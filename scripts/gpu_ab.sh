#!/bin/bash
# A/B of allocator flag sets on the microbench step: bash scripts/gpu_ab.sh "0 128" [reps]
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
rm -f gpurun_out/ab.log
for rep in $(seq 1 ${2:-3}); do
  for f in $1; do timeout -s KILL 120 python scripts/prof_mb.py $f 5 1 >> gpurun_out/ab.log 2>&1; done
done
