# tests + smoke + default bench (no CPU baseline) + solver sweep
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1200 python -m pytest tests/ -q -m gpu -x --timeout 600 2>&1 | tail -40 > gpurun_out/gpu_tests.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/gpu_smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/gpu_smoke.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_iter.log 2>&1
echo "bench exit $?" >> gpurun_out/bench_iter.log
timeout 600 python bench_solver.py --nodes 1024 4096 16384 --reps 5 > gpurun_out/solver_iter.log 2>&1
echo "solver exit $?" >> gpurun_out/solver_iter.log
