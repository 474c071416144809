mkdir -p gpurun_out
: > gpurun_out/multi_grid.txt
for S in 8 16; do
  for G in 18 37 74; do
    DS_PCG_GRID=$G timeout 900 python bench.py --sequences $S --steps 30 --warmup 3 > gpurun_out/mg.log 2>&1
    echo "S=$S G=$G $(grep '^{' gpurun_out/mg.log | cut -c30-60)" >> gpurun_out/multi_grid.txt
  done
done
