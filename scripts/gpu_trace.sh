mkdir -p gpurun_out
DS_PCG_TRACE=1 timeout 300 python scripts/pcg_iters.py > gpurun_out/pcg_trace.log 2>&1
