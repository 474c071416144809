# warp-per-chunk assembly v2 (staged, pixel-sorted segments, in-kernel finish)
mkdir -p gpurun_out/c44
timeout 900 python -m pytest tests/test_gpu_stages.py tests/test_gpu_baseline_parity.py tests/test_gpu_solve_fusion.py -q > gpurun_out/c44/tests.log 2>&1
echo "tests exit $?" >> gpurun_out/c44/tests.log
bash scripts/gpu_ab_env.sh DS_ASM=0 DS_ASM=1
cp gpurun_out/ab_summary.txt gpurun_out/c44/ab.txt
export DS_HOST_LM=1
DS_ASM=1 timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on \
      -k regex:"^k_assemble_warp" -s 1 -c 1 -o gpurun_out/c44/cfg2_k_assemble_warp -f python scripts/profile_frames.py 20 2 > gpurun_out/c44/ncu_1.log 2>&1
