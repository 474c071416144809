mkdir -p gpurun_out/c56
export DS_HOST_LM=1
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on \
      -k regex:"^k_tile_(assemble|finish)" -s 0 -c 2 -o gpurun_out/c56/cfg2_tiles -f python scripts/profile_frames.py 20 2 > gpurun_out/c56/ncu.log 2>&1
python scripts/tile_stats.py > gpurun_out/c56/tile_stats.log 2>&1
