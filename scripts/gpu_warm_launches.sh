mkdir -p gpurun_out
CMD="python scripts/profile_frames.py 40 2 cfg2"
$CMD > gpurun_out/warm_plain.log 2>&1 || exit 1
DS_HOST_LM=1 $CMD >> gpurun_out/warm_plain.log 2>&1 || exit 1
DS_HOST_LM=1 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
    --log-file gpurun_out/launches_warm_cfg2.csv $CMD > gpurun_out/ncu_warm.log 2>&1
