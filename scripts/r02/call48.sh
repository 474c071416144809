# candidate transforms in the PCG epilogue (one launch fewer per LM attempt)
mkdir -p gpurun_out/c48
timeout 1200 python -m pytest tests/test_gpu_solve_fusion.py tests/test_gpu_baseline_parity.py tests/test_gpu_pcg.py tests/test_gpu_acceptance.py -q -x > gpurun_out/c48/tests.log 2>&1
echo "tests exit $?" >> gpurun_out/c48/tests.log
bash scripts/gpu_ab_env.sh DS_FUSE_INC=0 DS_FUSE_INC=1
cp gpurun_out/ab_summary.txt gpurun_out/c48/ab.txt
