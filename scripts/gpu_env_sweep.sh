# usage: gpu_env_sweep.sh VAR "v1 v2 ..." [bench args...]; interleaved twice
VAR=$1; VALS=$2; shift 2
mkdir -p gpurun_out
for rep in 1 2; do for v in $VALS; do
  env $VAR=$v python bench.py "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$VAR=$v', d['value'], d['ms_per_step'])"
done; done
