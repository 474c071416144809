mkdir -p gpurun_out/c82
DS_PCG_TRACE=1 timeout 600 python scripts/profile_frames.py 20 2 > gpurun_out/c82/trace.log 2>&1
