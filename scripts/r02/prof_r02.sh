# Round-2 profile set: plain run first, then ncu (launch list + full sets).
mkdir -p gpurun_out/prof2
CMD2="python scripts/profile_frames.py 20 2"
export DS_HOST_LM=1   # per-kernel launches (the device LM graph hides kernels from ncu)
$CMD2 > gpurun_out/prof2/plain_cfg2.log 2>&1 || exit 1
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/prof2/launches_cfg2.csv $CMD2 > gpurun_out/prof2/ncu_launches.log 2>&1
for k in k_energy k_assemble_chunks k_pcg k_assoc_pair_terms k_model_splat; do
  timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on \
      -k regex:"^$k" -s 2 -c 1 -o gpurun_out/prof2/cfg2_$k -f $CMD2 > gpurun_out/prof2/ncu_cfg2_$k.log 2>&1
done
