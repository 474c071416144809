timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r02_c39_tests.log 2>&1
timeout 900 python bench.py > gpurun_out/r02_c39_bench_default.log 2>&1
timeout 900 python bench.py --config cfg3 --steps 54 --warmup 5 --no-cpu-baseline > gpurun_out/r02_c39_cfg3.log 2>&1
timeout 900 python bench.py --config cfg1 --steps 4 --warmup 5 > gpurun_out/r02_c39_cfg1.log 2>&1
timeout 900 python bench.py --sequences 8 --steps 30 --warmup 5 > gpurun_out/r02_c39_cfg5.log 2>&1
