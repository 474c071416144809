mkdir -p gpurun_out
DS_TRACE_HOST=1 timeout 300 python scripts/screen_probe.py 12 > gpurun_out/trace_host.log 2>&1
timeout 900 python bench.py --no-cpu-baseline --steps 40 > gpurun_out/bench_devlm40.log 2>&1
DS_HOST_LM=1 timeout 900 python bench.py --no-cpu-baseline --steps 40 > gpurun_out/bench_hostlm40.log 2>&1
