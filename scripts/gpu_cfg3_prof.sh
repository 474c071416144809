mkdir -p gpurun_out
CMD="python scripts/profile_frames.py 20 2 cfg3"
DS_HOST_LM=1 $CMD > gpurun_out/cfg3_plain.log 2>&1 || exit 1
DS_HOST_LM=1 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_cfg3.csv $CMD > gpurun_out/ncu_cfg3.log 2>&1
python bench.py --config cfg3 --steps 30 --warmup 5 > gpurun_out/cfg3_bench.json 2> gpurun_out/cfg3_bench.err
