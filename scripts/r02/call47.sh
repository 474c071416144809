# k_skin_incremental weight-load deferral + register-resident screening entries
mkdir -p gpurun_out/c47
timeout 900 python -m pytest tests/test_gpu_solve_fusion.py tests/test_gpu_baseline_parity.py -q -x > gpurun_out/c47/tests.log 2>&1
echo "tests exit $?" >> gpurun_out/c47/tests.log
bash scripts/gpu_ab_libs.sh base cur
cp gpurun_out/ab_summary.txt gpurun_out/c47/ab.txt
export DS_HOST_LM=1
for k in k_screen k_skin_incremental; do
  timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on \
      -k regex:"^$k" -s 1 -c 1 -o gpurun_out/c47/cfg2_$k -f python scripts/profile_frames.py 20 2 > gpurun_out/c47/ncu_$k.log 2>&1
done
