# Steady-state full captures (cfg2 frames 40-41), one ncu pass per kernel.
mkdir -p gpurun_out
CMD="python scripts/profile_frames.py 40 2"
$CMD > gpurun_out/prof_plain.log 2>&1 || exit 1
for k in k_assemble_chunks k_pcg k_screen k_pair_terms k_pair_runs k_model_splat k_rigid_finalize; do
  timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on \
      -k regex:"$k" -s 2 -c 1 -o gpurun_out/full_$k -f $CMD > gpurun_out/ncu_$k.log 2>&1
done
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_r01c.csv $CMD > gpurun_out/ncu_launches.log 2>&1
