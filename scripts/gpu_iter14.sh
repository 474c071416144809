mkdir -p gpurun_out
timeout 1200 python -m pytest tests/ -q -m gpu -x --timeout 600 2>&1 | tail -30 > gpurun_out/gpu_tests.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_iter.log 2>&1
timeout 1200 python bench.py --config cfg3 --steps 40 --warmup 3 > gpurun_out/bench_cfg3.log 2>&1
