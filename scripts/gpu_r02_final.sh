#!/bin/bash
# Round-end evidence at the current build: ncu summaries of every bench workload
# (scripts/gpu_ncu_apps.sh), the launch list of one bench step, then the bench
# lines (default + reference arm) and the GPU test suite.  Copy gpurun_out/prof_r02/*
# and the logs into profiles/r02/ afterwards (scripts/collect_r02.sh).
R=${R:-r02}
mkdir -p gpurun_out/prof_${R}
bash scripts/gpu_ncu_apps.sh
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${R}_launches.csv \
  python bench.py --steps 1 --warmup 1 --launch-list > gpurun_out/ncu_launches.log 2>&1
# the bench must find the summaries in profiles/ (same source hash) on this box too
mkdir -p profiles/${R}
cp gpurun_out/prof_${R}/ncu_*.json profiles/${R}/
timeout -s KILL 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1
timeout -s KILL 300 python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/bench_ref.log 2>&1
python scripts/refresh_profiles.py ${R} gpurun_out/prof_${R} > gpurun_out/refresh.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout -s KILL 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
# the extra full-length variants (bit mirror, all-tiled GoL; Wa-Tor against the live oracle and the static baseline)
DSR_FULL=1 timeout -s KILL 1500 python -m pytest tests/test_gpu_fulllength.py -q -p no:cacheprovider --durations=10 -s > gpurun_out/fulllength.log 2>&1
echo "pytest exit $?" >> gpurun_out/fulllength.log
