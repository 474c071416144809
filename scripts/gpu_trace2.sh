mkdir -p gpurun_out
DS_PCG_TRACE=1 timeout 300 python scripts/screen_probe.py 6 > gpurun_out/rigid_trace.log 2>&1
