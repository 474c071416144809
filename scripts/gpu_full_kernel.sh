# ncu --set full of kernels in a steady-state frame:
#   gpu_full_kernel.sh CONFIG NAME KERNEL_REGEX [COUNT] [SKIP_LAUNCHES] [SKIP_FRAMES]
mkdir -p gpurun_out
CFG=$1; NAME=$2; K=$3; CNT=${4:-1}; LS=${5:-0}; SKIP=${6:-40}
CMD="python scripts/profile_frames.py $SKIP 1 $CFG"
DS_HOST_LM=1 $CMD > gpurun_out/full_plain.log 2>&1 || exit 1
DS_HOST_LM=1 timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none \
    -k "regex:$K" --launch-skip $LS -c $CNT -o gpurun_out/${CFG}_$NAME -f $CMD > gpurun_out/ncu_full_$NAME.log 2>&1
