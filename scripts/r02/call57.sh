# tile assembly v2 (8-lane record groups from shared memory): parity, A/B, ncu
mkdir -p gpurun_out/c57
timeout 900 python -m pytest tests/test_gpu_stages.py -q -k "normal_equations or tile_assembly or pcg" > gpurun_out/c57/tests.log 2>&1
echo "exit $?" >> gpurun_out/c57/tests.log
: > gpurun_out/c57/ab.txt
for r in 1 2; do
  for v in "t3 DS_ASM_TILES=0" "t3 DS_ASM_TILES=1" "t2 DS_ASM_TILES=1"; do
    set -- $v
    env $2 DS_LIB_PATH=$PWD/ab/$1.so timeout 900 python bench.py --no-cpu-baseline --steps 60 > gpurun_out/c57/run.log 2>&1
    echo "$v run$r $(grep '^{' gpurun_out/c57/run.log | cut -c30-60) $(grep '^{' gpurun_out/c57/run.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["kernels"]["block_assembly"]["mean_launch_us"], d["kernels"]["reduce"]["mean_launch_us"], d["kernels"]["pattern"]["mean_launch_us"])')" >> gpurun_out/c57/ab.txt
  done
done
export DS_HOST_LM=1
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on \
      -k regex:"^k_tile_(assemble|finish|build)" -s 0 -c 3 -o gpurun_out/c57/cfg2_tiles -f python scripts/profile_frames.py 20 2 > gpurun_out/c57/ncu.log 2>&1
