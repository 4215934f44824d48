mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout -s KILL 1800 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider --durations=15 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout -s KILL 300 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1
timeout -s KILL 300 python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/bench_ref.log 2>&1
