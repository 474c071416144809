mkdir -p gpurun_out
./scripts/microbench/cond_test > gpurun_out/cond_test.log 2>&1
timeout 1200 python -m pytest tests/ -q -m gpu -x --timeout 600 2>&1 | tail -30 > gpurun_out/gpu_tests.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_iter.log 2>&1
DS_HOST_LM=1 timeout 900 python bench.py --no-cpu-baseline --steps 40 > gpurun_out/bench_hostlm.log 2>&1
