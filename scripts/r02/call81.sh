# final launch list (ncu, gpu__time_duration per launch) and PCG full set on the final build
mkdir -p gpurun_out/c81
CMD2="python scripts/profile_frames.py 20 2"
export DS_HOST_LM=1
$CMD2 > gpurun_out/c81/plain.log 2>&1 || exit 1
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/c81/launches_cfg2.csv $CMD2 > gpurun_out/c81/ncu_launches.log 2>&1
for k in k_pcg k_energy; do
  timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on \
      -k regex:"^$k" -s 2 -c 1 -o gpurun_out/c81/cfg2_$k -f $CMD2 > gpurun_out/c81/ncu_$k.log 2>&1
done
