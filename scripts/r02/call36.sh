timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r02_c36_tests.log 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02_c36_bench.log 2>&1
timeout 300 python bench_solver.py --nodes 16384 --reps 10 > gpurun_out/r02_c36_solver.log 2>&1
