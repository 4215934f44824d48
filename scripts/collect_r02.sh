#!/bin/bash
# after scripts/gpu_r02_final.sh: copy the evidence into the tracked profiles/r02/
set -e
P=profiles/r02
cp gpurun_out/prof_r02/* $P/
cp gpurun_out/bench.log $P/bench_full.log
grep '^{' gpurun_out/bench_ref.log | tail -1 > $P/bench_reference.json
cp gpurun_out/pytest_gpu.log $P/pytest_gpu.log
cp gpurun_out/smoke.log $P/smoke.log
cp gpurun_out/build_info.txt $P/ncu_build_info.txt
cp gpurun_out/fulllength.log $P/fulllength.log 2>/dev/null || true
