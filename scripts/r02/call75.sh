# config 5 sweep: independent config-2 sequences per GPU
mkdir -p gpurun_out/c75
for S in 8 16 32; do
  timeout 1200 python bench.py --sequences $S --steps 30 --no-cpu-baseline > gpurun_out/c75/bench_s$S.json 2>&1
done
nvidia-smi --query-gpu=memory.used,memory.total --format=csv > gpurun_out/c75/mem.txt
