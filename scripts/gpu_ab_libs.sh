# A/B of library builds under ab/: gpu_ab_libs.sh name1 name2 ...
mkdir -p gpurun_out
: > gpurun_out/ab_summary.txt
for r in 1 2; do
  for v in "$@"; do
    DS_LIB_PATH=$PWD/ab/$v.so timeout 900 python bench.py --no-cpu-baseline --steps 60 > gpurun_out/ab_run.log 2>&1
    echo "$v run$r $(grep '^{' gpurun_out/ab_run.log | cut -c30-60)" >> gpurun_out/ab_summary.txt
  done
done
