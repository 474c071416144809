# ncu --set full of one kernel in a steady-state frame: gpu_full_kernel.sh CONFIG KERNEL_REGEX [SKIP]
mkdir -p gpurun_out
CFG=$1; K=$2; SKIP=${3:-40}
CMD="python scripts/profile_frames.py $SKIP 1 $CFG"
DS_HOST_LM=1 $CMD > gpurun_out/full_plain.log 2>&1 || exit 1
DS_HOST_LM=1 timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:$K -c 1 \
    -o gpurun_out/${CFG}_$K -f $CMD > gpurun_out/ncu_full_$K.log 2>&1
