# the solve report kernel inside the device-LM graph (one host sync fewer per frame)
mkdir -p gpurun_out/c70
timeout 1200 python -m pytest tests/test_gpu_solve_fusion.py tests/test_gpu_baseline_parity.py tests/test_gpu_acceptance.py -q > gpurun_out/c70/tests.log 2>&1
echo "exit $?" >> gpurun_out/c70/tests.log
bash scripts/gpu_ab_libs.sh base rep
cp gpurun_out/ab_summary.txt gpurun_out/c70/ab.txt
