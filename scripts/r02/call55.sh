# surfel-tile block assembly (k_tiles.cu): parity, A/B vs record chunks, ncu
mkdir -p gpurun_out/c55
timeout 900 python -m pytest tests/test_gpu_stages.py tests/test_gpu_baseline_parity.py -q > gpurun_out/c55/tests.log 2>&1
echo "exit $?" >> gpurun_out/c55/tests.log
timeout 900 python -m pytest tests/test_gpu_solve_fusion.py tests/test_gpu_acceptance.py tests/test_gpu_pcg.py -q > gpurun_out/c55/tests2.log 2>&1
echo "exit $?" >> gpurun_out/c55/tests2.log
bash scripts/gpu_ab_env.sh DS_ASM_TILES=0 DS_ASM_TILES=1
cp gpurun_out/ab_summary.txt gpurun_out/c55/ab.txt
grep '^{' gpurun_out/ab_run.log > gpurun_out/c55/last.json
export DS_HOST_LM=1
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on \
      -k regex:"^k_tile_" -s 0 -c 4 -o gpurun_out/c55/cfg2_tiles -f python scripts/profile_frames.py 20 2 > gpurun_out/c55/ncu.log 2>&1
