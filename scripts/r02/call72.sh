# warp-field extension over device-side counts: no host sync between compaction and the greedy pass
mkdir -p gpurun_out/c72
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/c72/tests.log 2>&1
echo "exit $?" >> gpurun_out/c72/tests.log
bash scripts/gpu_ab_libs.sh base fus
cp gpurun_out/ab_summary.txt gpurun_out/c72/ab.txt
