mkdir -p gpurun_out/c61
timeout 900 python scripts/r02/cfg3_frames.py cfg3 > gpurun_out/c61/cfg3_frames.log 2>&1
