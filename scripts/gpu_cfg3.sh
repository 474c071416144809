mkdir -p gpurun_out
timeout 1200 python bench.py --config cfg3 --steps 40 --warmup 3 > gpurun_out/bench_cfg3.log 2>&1
echo "exit $?" >> gpurun_out/bench_cfg3.log
