#!/bin/bash
# GoL tiled-prepare A/B: GoL GPU tests at the in-tree build, then ab_gol.py per library ("-" = in-tree), and
# the per-pass ncu durations of the in-tree build:  bash scripts/gpu_ab_gol2.sh tag reps lib1.so ...
T=$1; R=$2; shift 2
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$T.log 2>&1
timeout -s KILL 1200 python -m pytest tests/test_gpu_gol.py tests/test_gpu_apps.py -q -x -m gpu -k "gol or life" --timeout 600 -p no:cacheprovider > gpurun_out/pytest_$T.log 2>&1
echo "pytest rc $?" >> gpurun_out/pytest_$T.log
out=gpurun_out/abg_$T.log; rm -f $out
for rep in $(seq 1 $R); do
  for lib in "$@"; do
    echo "LIB $lib" >> $out
    if [ "$lib" = "-" ]; then timeout -s KILL 300 python scripts/ab_gol.py 3 >> $out 2>&1
    else DSR_LIBPATH=$lib timeout -s KILL 300 python scripts/ab_gol.py 3 >> $out 2>&1; fi
  done
done
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_gol_tile_prepare" -s 4 -c 4 --csv python scripts/prof_targets.py gol16k-tiled > gpurun_out/ncu_$T.csv 2>&1
