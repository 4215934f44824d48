#!/bin/bash
# ncu --set full summaries of every bench workload at the current build (tagged with its
# source hash, so bench.py attaches their DRAM traffic to the roofline objects):
#   profiles/<R>/ncu_summary.json      microbench: k_mb_new_bulk (new1 + new4), k_mb_reduce x3, free passes
#   profiles/<R>/ncu_gol16k-tiled.json GoL 16384^2 (tiled prepare), one generation's 4 passes
#   profiles/<R>/ncu_gol16k.json       GoL 16384^2 (block list), 4 passes
#   profiles/<R>/ncu_gol16k-bits.json  GoL 16384^2 (alive-bit mirror), 4 passes
#   profiles/<R>/ncu_wator.json        Wa-Tor 2048^2, one step's 8 do-all bodies
#   profiles/<R>/ncu_nbody.json        N-body 65536, one step's kernels
# Output goes to gpurun_out/prof_<R>/ (copy into profiles/<R>/ after the call).
R=${R:-r02}
O=gpurun_out/prof_${R}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
python scripts/prof_targets.py none > /dev/null 2>&1    # writes gpurun_out/build_info.txt
NCU="ncu --set full --import-source on --clock-control none --kernel-name-base demangled"
cap() {   # name regex skip count target [source]
  timeout -s KILL 1500 $NCU -k regex:"$2" -s $3 -c $4 -o gpurun_out/${R}_$1 -f python scripts/prof_targets.py $5 > gpurun_out/ncu_$1.log 2>&1
}
cap mb_new "k_mb_new" 2 2 mb
cap mb_reduce "k_mb_reduce" 6 3 mb
cap mb_free "MbFree" 6 6 mb
python scripts/ncu_summarize.py $O/ncu_summary.json gpurun_out/${R}_mb_new.ncu-rep gpurun_out/${R}_mb_reduce.ncu-rep gpurun_out/${R}_mb_free.ncu-rep > $O/ncu_summary.txt
ncu -i gpurun_out/${R}_mb_new.ncu-rep --page source --csv --print-source cuda,sass > $O/mb_new_source.csv 2>/dev/null
for v in gol16k-tiled gol16k gol16k-bits; do
  cap $v "k_gol_tile|GolCand|GolAlive" 4 4 $v
  python scripts/ncu_summarize.py $O/ncu_$v.json gpurun_out/${R}_$v.ncu-rep > $O/ncu_$v.txt
done
ncu -i gpurun_out/${R}_gol16k-tiled.ncu-rep --page source --csv --print-source cuda,sass > $O/gol16k-tiled_source.csv 2>/dev/null
cap wator "k_doall.*Wt|k_doall_quad.*Wt" 16 8 wator
python scripts/ncu_summarize.py $O/ncu_wator.json gpurun_out/${R}_wator.ncu-rep > $O/ncu_wator.txt
cap nbody "k_nb_force_part|k_nb_merge_part" 2 2 nbody
python scripts/ncu_summarize.py $O/ncu_nbody.json gpurun_out/${R}_nbody.ncu-rep > $O/ncu_nbody.txt
gzip -f $O/*_source.csv
rm -f gpurun_out/${R}_*.ncu-rep
