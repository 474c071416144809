mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_pcg.py -q -x 2>&1 | tail -3 > gpurun_out/gpu_tests.log
CMD="python bench_solver.py --nodes 16384 --reps 3"
$CMD > gpurun_out/cfg4_plain.log 2>&1
for v in rows2 tma; do
  DS_SPMV=$v timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --cache-control all \
      -k regex:"^k_bsr_spmv" -s 1 -c 2 $CMD > gpurun_out/ncu_spmv_$v.log 2>&1
  DS_SPMV=$v python -m pytest tests/test_gpu_pcg.py -q -x -k spmv 2>&1 | tail -2 >> gpurun_out/gpu_tests.log
done
