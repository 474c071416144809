# Round-end profile set (see profiles/README.md): plain runs first, then ncu.
mkdir -p gpurun_out/prof
CMD2="python scripts/profile_frames.py 40 2"
export DS_HOST_LM=1   # per-kernel launches (the device LM graph hides kernels from ncu)
$CMD2 > gpurun_out/prof/plain_cfg2.log 2>&1 || exit 1
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/prof/launches_cfg2.csv $CMD2 > gpurun_out/prof/ncu_launches.log 2>&1
for k in k_assemble_chunks k_pcg k_assoc_pair_terms k_model_splat k_screen k_rigid_terms k_energy; do
  timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
      -k regex:"^$k" -s 2 -c 1 -o gpurun_out/prof/cfg2_$k -f $CMD2 > gpurun_out/prof/ncu_cfg2_$k.log 2>&1
done
CMD4="python bench_solver.py --nodes 16384 --reps 3"
$CMD4 > gpurun_out/prof/plain_cfg4.log 2>&1 || exit 1
for k in k_forward_warp k_bsr_spmv_rows k_assemble_chunks; do
  timeout 900 ncu --set full --clock-control none --cache-control all --import-source on \
      -k regex:"^$k\$" -s 1 -c 1 -o gpurun_out/prof/cfg4_$k -f $CMD4 > gpurun_out/prof/ncu_cfg4_$k.log 2>&1
done
