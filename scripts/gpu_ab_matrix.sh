# A/B matrix: gpu_ab_matrix.sh "lib:ENV=val ..." ...  (each arg = lib name under ab/ + env assignments)
mkdir -p gpurun_out
: > gpurun_out/ab_summary.txt
for r in 1 2; do
  for spec in "$@"; do
    lib=${spec%%:*}; envs=${spec#*:}; [ "$envs" = "$spec" ] && envs=""
    env $envs DS_LIB_PATH=$PWD/ab/$lib.so timeout 900 python bench.py --no-cpu-baseline --steps ${AB_STEPS:-60} ${AB_ARGS:-} > gpurun_out/ab_run.log 2>&1
    echo "$spec run$r $(grep '^{' gpurun_out/ab_run.log | cut -c30-60)" >> gpurun_out/ab_summary.txt
  done
done
