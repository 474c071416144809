# rigid ICP term kernel: two pixels per step (bit-identical sums); direct reference test
mkdir -p gpurun_out/c54
timeout 900 python -m pytest tests/test_gpu_baseline_parity.py tests/test_gpu_solve_fusion.py -q > gpurun_out/c54/tests.log 2>&1
echo "exit $?" >> gpurun_out/c54/tests.log
bash scripts/gpu_ab_libs.sh base cur
cp gpurun_out/ab_summary.txt gpurun_out/c54/ab.txt
grep '^{' gpurun_out/ab_run.log > gpurun_out/c54/last_cur.json
