mkdir -p gpurun_out/c62
timeout 900 python bench.py --config cfg3 --no-cpu-baseline > gpurun_out/c62/bench_cfg3.json 2>&1
timeout 900 python bench.py --config cfg1 > gpurun_out/c62/bench_cfg1.json 2>&1
