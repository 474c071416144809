# PCG: 256-thread CTAs and cp.async slice staging overlapped with the inverses
mkdir -p gpurun_out/c64
DS_LIB_PATH=$PWD/ab/p256a.so timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/c64/tests.log 2>&1
echo "exit $?" >> gpurun_out/c64/tests.log
: > gpurun_out/c64/ab.txt
for r in 1 2; do
  for v in p512 pasync p256 p256a; do
    DS_LIB_PATH=$PWD/ab/$v.so timeout 900 python bench.py --no-cpu-baseline --steps 60 > gpurun_out/c64/run.log 2>&1
    echo "$v run$r $(grep '^{' gpurun_out/c64/run.log | cut -c30-60) $(grep '^{' gpurun_out/c64/run.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["kernels"]["pcg"]["mean_launch_us"])')" >> gpurun_out/c64/ab.txt
  done
done
