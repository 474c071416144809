# multi-chunk JtJ blocks finished inside k_assemble_chunks (no k_assemble_finish launch)
mkdir -p gpurun_out/c49
timeout 1200 python -m pytest tests/test_gpu_stages.py tests/test_gpu_baseline_parity.py tests/test_gpu_solve_fusion.py tests/test_gpu_acceptance.py -q -x > gpurun_out/c49/tests.log 2>&1
echo "tests exit $?" >> gpurun_out/c49/tests.log
bash scripts/gpu_ab_env.sh DS_ASM_FINISH=1 DS_ASM_FINISH=0
cp gpurun_out/ab_summary.txt gpurun_out/c49/ab.txt
