#!/bin/bash
# Round-end evidence: launch list of one bench step, ncu --set full of the step's kernels,
# the bench lines (microbench + apps).  Everything lands in gpurun_out/.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
NCU="ncu --set full --import-source on --clock-control none --kernel-name-base demangled"
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_launches.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1
timeout -s KILL 600 $NCU -k regex:"k_mb_new" -s 2 -c 1 -o gpurun_out/r01_mb_new -f python scripts/prof_targets.py mb > gpurun_out/ncu_a.log 2>&1
timeout -s KILL 600 $NCU -k regex:"k_mb_reduce" -s 6 -c 3 -o gpurun_out/r01_mb_reduce -f python scripts/prof_targets.py mb > gpurun_out/ncu_b.log 2>&1
timeout -s KILL 600 $NCU -k regex:"MbFree" -s 6 -c 6 -o gpurun_out/r01_mb_free -f python scripts/prof_targets.py mb > gpurun_out/ncu_c.log 2>&1
timeout -s KILL 600 $NCU -k regex:"k_compact" -s 13 -c 3 -o gpurun_out/r01_compact -f python scripts/prof_targets.py mb > gpurun_out/ncu_d.log 2>&1
timeout -s KILL 600 $NCU -k regex:"k_nb_|NbMove|NbSnapshot" -s 8 -c 6 -o gpurun_out/r01_nbody -f python scripts/prof_targets.py nbody > gpurun_out/ncu_e.log 2>&1
timeout -s KILL 600 $NCU -k regex:"Wt" -s 8 -c 8 -o gpurun_out/r01_wator -f python scripts/prof_targets.py wator > gpurun_out/ncu_f.log 2>&1
timeout -s KILL 1200 $NCU -k regex:"Gol(CandPrepare|AliveUpdate|CandUpdate|AlivePrepare)" -s 4 -c 4 -o gpurun_out/r01_gol16k -f python scripts/prof_targets.py gol16k > gpurun_out/ncu_g.log 2>&1
timeout -s KILL 300 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1
rm -f gpurun_out/bench_apps.log
for w in wator gol gol16k gol16k-bits nbody; do
  timeout -s KILL 300 python bench.py --workload $w --steps 10 --warmup 3 >> gpurun_out/bench_apps.log 2>&1
done
timeout -s KILL 600 python scripts/prof_apps.py > gpurun_out/prof_apps.log 2>&1
# summaries travel back (gpurun_out is capped at 64 MiB): per-line source pages of the
# allocation kernel and the GoL passes, then drop the big reports
python scripts/refresh_profiles.py r01 gpurun_out/prof_r01 > gpurun_out/refresh.log 2>&1
ncu -i gpurun_out/r01_mb_new.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/prof_r01/mb_new_source.csv 2>/dev/null
ncu -i gpurun_out/r01_gol16k.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/prof_r01/gol16k_source.csv 2>/dev/null
gzip -f gpurun_out/prof_r01/*_source.csv
rm -f gpurun_out/r01_gol16k.ncu-rep gpurun_out/r01_nbody.ncu-rep gpurun_out/r01_wator.ncu-rep gpurun_out/r01_compact.ncu-rep gpurun_out/r01_mb_free.ncu-rep
