# Plain run first (must exit 0), then the ncu launch list and a full capture of
# the top kernels (B200_PROFILING.md recipe). Outputs land in gpurun_out/.
mkdir -p gpurun_out
CMD="python bench.py --steps 4 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/ncu_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on \
    -k regex:"k_screen|k_assemble_chunks|k_pcg|k_forward_warp_list|k_model_splat|k_pair_terms|k_greedy_nodes|k_sort_lists" \
    -s 800 -c 12 -o gpurun_out/prof_full $CMD > gpurun_out/ncu_full.log 2>&1
for g in 37 74 148; do
  DS_PCG_GRID=$g timeout 600 python bench.py --steps 40 --no-cpu-baseline > gpurun_out/sweep_pcg_$g.log 2>&1
done
