mkdir -p gpurun_out/c69
timeout 600 python scripts/r02/host_trace.py > gpurun_out/c69/host_trace.log 2>&1
