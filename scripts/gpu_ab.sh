# A/B timing of two library builds on the same box, interleaved
mkdir -p gpurun_out
for r in 1 2; do
  for v in A B; do
    DS_LIB_PATH=$PWD/ab/lib$v.so timeout 900 python bench.py --no-cpu-baseline --steps 60 > gpurun_out/ab_${v}_$r.log 2>&1
  done
done
for f in gpurun_out/ab_*.log; do echo "$f $(grep '^{' $f | cut -c30-60)"; done > gpurun_out/ab_summary.txt
