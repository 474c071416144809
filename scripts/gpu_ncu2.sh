# Steady-state profile of cfg2 frames 40-41: plain run, launch list, full capture.
mkdir -p gpurun_out
CMD="python scripts/profile_frames.py 40 2"
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_r01b.csv $CMD > gpurun_out/ncu_launches.log 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:"k_screen|k_assemble_chunks|k_pcg|k_model_splat|k_pair_terms|k_sort_lists|k_rigid_terms|k_scan" \
    -c 16 -o gpurun_out/prof_full_r01b -f $CMD > gpurun_out/ncu_full.log 2>&1
