#!/bin/bash
# A/B: drain block-mapped vs quad (flag), odd-free block (variant oddb), GoL selective do-all vs not (variant nosel)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout -s KILL 900 python -m pytest tests/test_gpu_gol.py tests/test_gpu_allocator.py -q -x -p no:cacheprovider > gpurun_out/ab_pytest.log 2>&1
rm -f gpurun_out/ab2.log
for v in default oddb; do
  lib=""; [ "$v" != default ] && lib=paper_1810_11765_b200/_build/libdsr_$v.so
  echo "variant $v" >> gpurun_out/ab2.log
  DSR_LIBPATH=$lib timeout -s KILL 200 python scripts/mb_variants.py 5 bulk,quad_drain >> gpurun_out/ab2.log 2>&1
done
for v in default nosel; do
  lib=""; [ "$v" != default ] && lib=paper_1810_11765_b200/_build/libdsr_$v.so
  echo "variant $v" >> gpurun_out/ab2.log
  DSR_LIBPATH=$lib timeout -s KILL 300 python scripts/gol_variants.py 3 >> gpurun_out/ab2.log 2>&1
done
