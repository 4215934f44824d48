#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout -s KILL 1200 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:"Gol(CandPrepare|AliveUpdate|CandUpdate|AlivePrepare)" -s 4 -c 4 -o gpurun_out/r01_gol16k -f python scripts/prof_targets.py gol16k > gpurun_out/ncu_gol.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_gol.log
