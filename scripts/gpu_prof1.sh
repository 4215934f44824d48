#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
N="ncu --set full --import-source on --clock-control none"
timeout -s KILL 600 $N -k regex:k_mb_new -s 2 -c 1 -o gpurun_out/r01_mb_new python scripts/prof_targets.py mb > gpurun_out/ncu1.log 2>&1
timeout -s KILL 600 $N -k regex:k_mb_reduce -s 6 -c 6 -o gpurun_out/r01_mb_reduce python scripts/prof_targets.py mb > gpurun_out/ncu2.log 2>&1
timeout -s KILL 600 $N -k regex:"MbFreeAll|k_compact" -s 4 -c 2 -o gpurun_out/r01_mb_free python scripts/prof_targets.py mb > gpurun_out/ncu3.log 2>&1
timeout -s KILL 600 $N -k regex:"k_nb_force_part|k_nb_merge_part" -s 2 -c 2 -o gpurun_out/r01_nbody python scripts/prof_targets.py nbody > gpurun_out/ncu4.log 2>&1
timeout -s KILL 900 $N -k regex:"k_doall" -s 8 -c 4 -o gpurun_out/r01_gol16k python scripts/prof_targets.py gol16k > gpurun_out/ncu5.log 2>&1
timeout -s KILL 600 $N -k regex:"k_doall" -s 16 -c 8 -o gpurun_out/r01_wator python scripts/prof_targets.py wator > gpurun_out/ncu6.log 2>&1
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
