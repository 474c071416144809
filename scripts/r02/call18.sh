timeout 300 python -m pytest tests/test_gpu_solve_fusion.py tests/test_gpu_stages.py tests/test_gpu_baseline_parity.py -q -x > gpurun_out/r02_c18_tests.log 2>&1
DS_TRACE_HOST=1 timeout 120 python scripts/r02/gn_probe.py cfg2 22 pcg10 > gpurun_out/r02_c18_trace.log 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02_c18_bench.log 2>&1
