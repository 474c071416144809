# splat pass 1 with the fused warp: lane 0 warps, 2 / 4 lanes share the disk (shuffled live state)
mkdir -p gpurun_out/c76
for v in sh2 sh4; do
  DS_LIB_PATH=$PWD/ab/$v.so timeout 900 python -m pytest tests/test_gpu_stages.py tests/test_gpu_baseline_parity.py -q -x > gpurun_out/c76/tests_$v.log 2>&1
  echo "exit $?" >> gpurun_out/c76/tests_$v.log
done
bash scripts/gpu_ab_libs.sh base sh2 sh4
cp gpurun_out/ab_summary.txt gpurun_out/c76/ab.txt
