#!/bin/bash
# microbench bulk work-unit sweep (variant libraries through DSR_LIBPATH) + ncu of the bulk kernel
mkdir -p gpurun_out
python -c "from paper_1810_11765_b200 import build; build.build()
for u in (3072, 6144):
    build.build(variant=f'unit{u}', defines=[f'DSR_MB_UNIT={u}'])"
timeout 300 python scripts/mb_variants.py 5 bulk > gpurun_out/mbv.log 2>&1
for u in 3072 6144; do DSR_LIBPATH=paper_1810_11765_b200/_build/libdsr_unit$u.so timeout 120 python scripts/mb_variants.py 5 bulk >> gpurun_out/mbv.log 2>&1; done
timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:k_mb_new_bulk -s 2 -c 2 -o gpurun_out/r02_mb_bulk -f python scripts/prof_targets.py mb > gpurun_out/ncu1.log 2>&1
timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:k_doall_quad -s 6 -c 6 -o gpurun_out/r02_mb_quad -f python scripts/prof_targets.py mb > gpurun_out/ncu2.log 2>&1
