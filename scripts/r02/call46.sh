# warp assembly v3: resident grid with warps striding over chunks
mkdir -p gpurun_out/c46
timeout 900 python -m pytest tests/test_gpu_stages.py tests/test_gpu_baseline_parity.py -q -x > gpurun_out/c46/tests.log 2>&1
echo "tests exit $?" >> gpurun_out/c46/tests.log
bash scripts/gpu_ab_env.sh DS_ASM=0 DS_ASM=1 DS_ASM_CTAS=2
cp gpurun_out/ab_summary.txt gpurun_out/c46/ab.txt
export DS_HOST_LM=1
DS_ASM=1 timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on \
      -k regex:"^k_assemble_warp" -s 1 -c 1 -o gpurun_out/c46/cfg2_k_assemble_warp -f python scripts/profile_frames.py 20 2 > gpurun_out/c46/ncu_1.log 2>&1
DS_ASM=0 timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on \
      -k regex:"^k_assemble_chunks" -s 1 -c 1 -o gpurun_out/c46/cfg2_k_assemble_chunks -f python scripts/profile_frames.py 20 2 > gpurun_out/c46/ncu_0.log 2>&1
