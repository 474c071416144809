mkdir -p gpurun_out
timeout 1200 python -m pytest tests/ -q -m gpu -x --timeout 600 2>&1 | tail -30 > gpurun_out/gpu_tests.log
timeout 600 python bench_solver.py --nodes 1024 4096 8192 16384 --reps 5 > gpurun_out/solver_iter.log 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_iter.log 2>&1
