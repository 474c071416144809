# per-kernel warm durations for several libs: gpu_ab_kernels.sh lib1 lib2 ...
mkdir -p gpurun_out
for v in "$@"; do
  DS_LIB_PATH=$PWD/ab/$v.so DS_HOST_LM=1 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
    --log-file gpurun_out/abk_$v.csv python scripts/profile_frames.py 40 2 cfg2 > gpurun_out/abk_$v.log 2>&1
done
