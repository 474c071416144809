mkdir -p gpurun_out/prof3
CMD2="python scripts/profile_frames.py 20 2"
export DS_HOST_LM=1
$CMD2 > gpurun_out/prof3/plain.log 2>&1 || exit 1
for k in k_screen k_skin_incremental; do
  timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on \
      -k regex:"^$k" -s 1 -c 1 -o gpurun_out/prof3/cfg2_$k -f $CMD2 > gpurun_out/prof3/ncu_$k.log 2>&1
done
