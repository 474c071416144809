# warp-per-chunk assembly: parity tests, A/B against the round-1 kernel, ncu
mkdir -p gpurun_out/c43
timeout 900 python -m pytest tests/test_gpu_stages.py tests/test_gpu_baseline_parity.py -q -x > gpurun_out/c43/tests.log 2>&1
echo "tests exit $?" >> gpurun_out/c43/tests.log
bash scripts/gpu_ab_env.sh DS_ASM=0 DS_ASM=1
cp gpurun_out/ab_summary.txt gpurun_out/c43/ab.txt
export DS_HOST_LM=1
for m in 0 1; do
  k=k_assemble_warp; [ $m = 0 ] && k=k_assemble_chunks
  DS_ASM=$m timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on \
      -k regex:"^$k" -s 1 -c 1 -o gpurun_out/c43/cfg2_$k -f python scripts/profile_frames.py 20 2 > gpurun_out/c43/ncu_$m.log 2>&1
done
