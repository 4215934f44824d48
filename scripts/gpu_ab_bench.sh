mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout -s KILL 600 python -m pytest tests -q -x -m gpu -k "probe or torture or replay or microbench or wator_every or gol_every or compact" --timeout 300 -p no:cacheprovider > gpurun_out/pytest_sub.log 2>&1
bash scripts/gpu_ab_lib.sh paper_1810_11765_b200/_build/libdsr_base.so 3
timeout -s KILL 300 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1
