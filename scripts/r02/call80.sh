# pair successors found in the segment by the assembly (no k_pair_next launch)
mkdir -p gpurun_out/c80
timeout 1200 python -m pytest tests/test_gpu_stages.py tests/test_gpu_baseline_parity.py tests/test_gpu_solve_fusion.py -q > gpurun_out/c80/tests.log 2>&1
echo "exit $?" >> gpurun_out/c80/tests.log
bash scripts/gpu_ab_env.sh DS_PAIR_NEXT=1 DS_PAIR_NEXT=0
cp gpurun_out/ab_summary.txt gpurun_out/c80/ab.txt
