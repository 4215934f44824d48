#!/bin/bash
# Round-2 first GPU pass: build, smoke, the -m gpu suite, the default bench line (with the apps
# block), the reference arm, the launch list of one bench step and ncu --set full of the
# allocation kernel.  Everything lands in gpurun_out/.
R=${R:-r02}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout -s KILL 1800 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider --durations=25 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout -s KILL 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1
timeout -s KILL 300 python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/bench_ref.log 2>&1
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${R}_launches.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-apps > gpurun_out/ncu_launches.log 2>&1
NCU="ncu --set full --import-source on --clock-control none --kernel-name-base demangled"
timeout -s KILL 600 $NCU -k regex:"k_mb_new" -s 2 -c 2 -o gpurun_out/${R}_mb_new -f python scripts/prof_targets.py mb > gpurun_out/ncu_a.log 2>&1
timeout -s KILL 600 $NCU -k regex:"k_mb_reduce" -s 6 -c 3 -o gpurun_out/${R}_mb_reduce -f python scripts/prof_targets.py mb > gpurun_out/ncu_b.log 2>&1
timeout -s KILL 600 $NCU -k regex:"MbFree" -s 6 -c 6 -o gpurun_out/${R}_mb_free -f python scripts/prof_targets.py mb > gpurun_out/ncu_c.log 2>&1
python scripts/refresh_profiles.py ${R} gpurun_out/prof_${R} > gpurun_out/refresh.log 2>&1
ncu -i gpurun_out/${R}_mb_new.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/prof_${R}/mb_new_source.csv 2>/dev/null
gzip -f gpurun_out/prof_${R}/*_source.csv
rm -f gpurun_out/${R}_mb_reduce.ncu-rep gpurun_out/${R}_mb_free.ncu-rep
