set -x
mkdir -p gpurun_out
(nproc; lscpu | head -25; free -g) > gpurun_out/r02_c1_host.txt 2>&1
timeout 300 python -m pytest tests -m gpu -x -q > gpurun_out/r02_c1_tests.log 2>&1
timeout 400 python scripts/r02/gn_probe.py cfg2 26 > gpurun_out/r02_c1_gn_cfg2.log 2>&1
timeout 200 python scripts/r02/gn_probe.py cfg1 10 > gpurun_out/r02_c1_gn_cfg1.log 2>&1
timeout 400 python scripts/r02/lockstep_probe.py cfg1 > gpurun_out/r02_c1_lock_cfg1.log 2>&1
timeout 400 python scripts/r02/lockstep_probe.py cfg2 3 > gpurun_out/r02_c1_lock_cfg2.log 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02_c1_bench.log 2>&1
tail -3 gpurun_out/r02_c1_tests.log
