mkdir -p gpurun_out/c79
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/c79/tests.log 2>&1
echo "exit $?" >> gpurun_out/c79/tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/c79/smoke.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/c79/bench_20.json 2>&1
timeout 1200 python bench.py > gpurun_out/c79/bench_default.json 2>&1
