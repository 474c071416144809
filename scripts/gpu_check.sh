mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1200 python -m pytest tests/ -q -m gpu -x --timeout 600 2>&1 | tail -60 > gpurun_out/gpu_tests.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/gpu_smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/gpu_smoke.log
