mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_pcg.py -q -x --timeout 600 2>&1 | tail -5 > gpurun_out/gpu_tests.log
for S in 4 8 16; do
  timeout 900 python bench.py --sequences $S --steps 30 --warmup 3 > gpurun_out/multi_$S.log 2>&1
done
CMD="python bench_solver.py --nodes 16384 --reps 3"
$CMD > gpurun_out/cfg4_plain.log 2>&1
for v in rows tma; do
  DS_SPMV=$v timeout 600 ncu --set full --clock-control none --cache-control all \
      -k regex:"^k_bsr_spmv" -s 1 -c 1 -o gpurun_out/cfg4_spmv_$v -f $CMD > gpurun_out/ncu_spmv_$v.log 2>&1
done
timeout 600 ncu --set full --clock-control none --cache-control all \
      -k regex:"^k_forward_warp" -s 1 -c 1 -o gpurun_out/cfg4_fw2 -f $CMD > gpurun_out/ncu_fw2.log 2>&1
