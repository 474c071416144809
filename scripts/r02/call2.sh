mkdir -p gpurun_out
timeout 600 python scripts/r02/frame2_debug.py > gpurun_out/r02_c2_frame2.log 2>&1
timeout 400 python scripts/r02/lockstep_probe.py cfg1 > gpurun_out/r02_c2_lock_cfg1.log 2>&1
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02_c2_ref_cfg2.log 2>&1
timeout 600 python bench.py --impl reference --config cfg1 --steps 20 --warmup 5 > gpurun_out/r02_c2_ref_cfg1.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_c2_bench.log 2>&1
