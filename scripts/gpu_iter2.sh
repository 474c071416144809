mkdir -p gpurun_out
timeout 1200 python -m pytest tests/ -q -m gpu -x --timeout 600 2>&1 | tail -40 > gpurun_out/gpu_tests.log
timeout 120 ./scripts/microbench/gridsync > gpurun_out/gridsync.log 2>&1
timeout 300 python scripts/pcg_iters.py > gpurun_out/pcg_iters.log 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_iter.log 2>&1
echo "bench exit $?" >> gpurun_out/bench_iter.log
