mkdir -p gpurun_out
CMD="python scripts/profile_frames.py 20 1 cfg3"
DS_HOST_LM=1 $CMD > gpurun_out/cfg3_plain.log 2>&1 || exit 1
for k in k_screen k_node_edges_grid k_skin_incremental; do
DS_HOST_LM=1 timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:$k -c 1 \
    -o gpurun_out/cfg3_$k -f $CMD > gpurun_out/ncu_full_$k.log 2>&1
done
