#!/bin/bash
# One microbench iteration on the GPU box: build, allocator parity tests, A/B of
# the phase times against a saved library ($1), ncu of the new kernel.
#   bash scripts/gpu_iter_mb.sh path/to/base.so [tag]
mkdir -p gpurun_out
T=${2:-it}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$T.log 2>&1
timeout -s KILL 900 python -m pytest tests/test_gpu_allocator.py -q -x -m gpu --timeout 300 -p no:cacheprovider > gpurun_out/pytest_$T.log 2>&1
echo "pytest rc $?" >> gpurun_out/pytest_$T.log
bash scripts/gpu_ab_lib_mb.sh $1 3 > /dev/null 2>&1
cp gpurun_out/ab_lib.log gpurun_out/ab_$T.log
NCU="ncu --set full --import-source on --clock-control none --kernel-name-base demangled"
timeout -s KILL 600 $NCU -k regex:"k_mb_new" -s 2 -c 2 -o gpurun_out/${T}_mb_new -f python scripts/prof_targets.py mb > gpurun_out/ncu_$T.log 2>&1
python scripts/ncu_summarize.py gpurun_out/ncu_${T}.json gpurun_out/${T}_mb_new.ncu-rep > gpurun_out/ncu_${T}.txt 2>&1
ncu -i gpurun_out/${T}_mb_new.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/src_${T}.csv 2>/dev/null
gzip -f gpurun_out/src_${T}.csv
