mkdir -p gpurun_out
python scripts/compare_pipeline.py articulated_two_part 6 > gpurun_out/cmp_a2p.log 2>&1
python scripts/compare_pipeline.py rigid_orbit 6 >> gpurun_out/cmp_a2p.log 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench1.log 2>&1
echo "bench exit $?" >> gpurun_out/bench1.log
