mkdir -p gpurun_out
CMD="python bench_solver.py --nodes 16384 --reps 3"
$CMD > gpurun_out/cfg4_plain.log 2>&1
for v in rows rows2 rows3; do
  DS_SPMV=$v timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --cache-control all \
      -k regex:"^k_bsr_spmv" -s 1 -c 2 $CMD > gpurun_out/ncu_spmv_$v.log 2>&1
done
timeout 600 ncu --set full --clock-control none --cache-control all \
      -k k_forward_warp -s 1 -c 1 -o gpurun_out/cfg4_fwu2 -f $CMD > gpurun_out/ncu_fwu2.log 2>&1
