#!/bin/bash
mkdir -p gpurun_out
python -c "from paper_1810_11765_b200 import build; build.build()
for m in (4, 6):
    build.build(variant=f'minb{m}', defines=[f'DSR_DOALL_MINB={m}'])"
: > gpurun_out/minb.log
for lib in libdsr.so _build/libdsr_minb4.so _build/libdsr_minb6.so; do
  echo "== $lib" >> gpurun_out/minb.log
  DSR_LIBPATH=paper_1810_11765_b200/$lib timeout 300 python scripts/gol_variants.py 4 >> gpurun_out/minb.log 2>&1
  DSR_LIBPATH=paper_1810_11765_b200/$lib timeout 300 python scripts/ab_apps.py 0 wator >> gpurun_out/minb.log 2>&1
  DSR_LIBPATH=paper_1810_11765_b200/$lib timeout 300 python scripts/mb_variants.py 3 bulk >> gpurun_out/minb.log 2>&1
done
