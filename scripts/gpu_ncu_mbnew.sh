#!/bin/bash
R=${R:-r02}
mkdir -p gpurun_out/prof_${R}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
NCU="ncu --set full --import-source on --clock-control none --kernel-name-base demangled"
timeout -s KILL 900 $NCU -k regex:"k_mb_new" -s 2 -c 2 -o gpurun_out/${R}_mb_new -f python scripts/prof_targets.py mb > gpurun_out/ncu_a.log 2>&1
python scripts/ncu_summarize.py gpurun_out/prof_${R}/ncu_mbnew_only.json gpurun_out/${R}_mb_new.ncu-rep > gpurun_out/prof_${R}/ncu_mbnew_only.txt
ncu -i gpurun_out/${R}_mb_new.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/prof_${R}/mb_new_source.csv 2>/dev/null
gzip -f gpurun_out/prof_${R}/mb_new_source.csv
rm -f gpurun_out/${R}_mb_new.ncu-rep
