# A/B of one build under two environments, interleaved: gpu_ab_env.sh "VAR=a" "VAR=b"
mkdir -p gpurun_out
: > gpurun_out/ab_summary.txt
for r in 1 2; do
  for e in "$@"; do
    env $e timeout 900 python bench.py --no-cpu-baseline --steps 60 > gpurun_out/ab_run.log 2>&1
    echo "$e run$r $(grep '^{' gpurun_out/ab_run.log | cut -c30-60)" >> gpurun_out/ab_summary.txt
  done
done
