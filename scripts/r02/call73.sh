# solve graph captured while the rigid ICP runs (pose read from the device)
mkdir -p gpurun_out/c73
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/c73/tests.log 2>&1
echo "exit $?" >> gpurun_out/c73/tests.log
: > gpurun_out/c73/ab.txt
for r in 1 2; do
  for v in "fus DS_EARLY_GRAPH=1" "early DS_EARLY_GRAPH=0" "early DS_EARLY_GRAPH=1"; do
    set -- $v
    env $2 DS_LIB_PATH=$PWD/ab/$1.so timeout 900 python bench.py --no-cpu-baseline --steps 60 > gpurun_out/c73/run.log 2>&1
    echo "$v run$r $(grep '^{' gpurun_out/c73/run.log | cut -c30-60)" >> gpurun_out/c73/ab.txt
  done
done
