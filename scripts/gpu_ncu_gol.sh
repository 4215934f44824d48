#!/bin/bash
# ncu --set full of one GoL 16384^2 generation (variant $1: gol16k | gol16k-tiled | gol16k-tiledall | gol16k-bits)
V=${1:-gol16k-tiled}
R=${R:-r02}
mkdir -p gpurun_out/prof_${R}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
NCU="ncu --set full --import-source on --clock-control none --kernel-name-base demangled"
timeout -s KILL 1500 $NCU -k regex:"k_gol_tile|GolCand|GolAlive" -s 4 -c 4 -o gpurun_out/${R}_${V} -f python scripts/prof_targets.py $V > gpurun_out/ncu_gol.log 2>&1
python scripts/ncu_summarize.py gpurun_out/prof_${R}/ncu_${V}.json gpurun_out/${R}_${V}.ncu-rep > gpurun_out/prof_${R}/ncu_${V}.txt
ncu -i gpurun_out/${R}_${V}.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/prof_${R}/${V}_source.csv 2>/dev/null
gzip -f gpurun_out/prof_${R}/${V}_source.csv
rm -f gpurun_out/${R}_${V}.ncu-rep
