mkdir -p gpurun_out/c53
timeout 900 python -m pytest tests/test_gpu_baseline_parity.py -q -k "compiled_reference" > gpurun_out/c53/tests_gpu.log 2>&1
echo "exit $?" >> gpurun_out/c53/tests_gpu.log
