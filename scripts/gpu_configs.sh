mkdir -p gpurun_out
for S in 8 16 32; do
  timeout 900 python bench.py --sequences $S --steps 30 --warmup 3 > gpurun_out/multi_$S.log 2>&1
done
timeout 1200 python bench.py --config cfg3 --steps 40 --warmup 3 > gpurun_out/bench_cfg3.log 2>&1
timeout 600 python bench_solver.py --nodes 1024 4096 8192 16384 --reps 5 > gpurun_out/solver_iter.log 2>&1
