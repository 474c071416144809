# cfg4 (16k nodes, 2.1M surfels) full captures of the HBM-roofline kernels.
mkdir -p gpurun_out
CMD="python bench_solver.py --nodes 16384 --reps 3"
$CMD > gpurun_out/cfg4_plain.log 2>&1 || exit 1
for k in k_forward_warp k_bsr_spmv k_assemble_chunks k_pcg; do
  timeout 600 ncu --set full --clock-control none --import-source on --cache-control all \
      -k regex:"^$k" -s 1 -c 1 -o gpurun_out/cfg4_$k -f $CMD > gpurun_out/ncu_cfg4_$k.log 2>&1
done
