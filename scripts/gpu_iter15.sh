mkdir -p gpurun_out
timeout 1200 python -m pytest tests/ -q -m gpu -x --timeout 600 2>&1 | tail -30 > gpurun_out/gpu_tests.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_iter.log 2>&1
CMD="python scripts/profile_frames.py 40 2"
DS_HOST_LM=1 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_r01d.csv $CMD > gpurun_out/ncu_launches.log 2>&1
