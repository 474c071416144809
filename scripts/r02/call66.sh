mkdir -p gpurun_out/c66
: > gpurun_out/c66/ab.txt
for r in 1 2; do
  for v in p256a p256a2; do
    DS_LIB_PATH=$PWD/ab/$v.so timeout 900 python bench.py --no-cpu-baseline --steps 60 > gpurun_out/c66/run.log 2>&1
    echo "$v run$r $(grep '^{' gpurun_out/c66/run.log | cut -c30-60) $(grep '^{' gpurun_out/c66/run.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["kernels"]["pcg"]["mean_launch_us"])')" >> gpurun_out/c66/ab.txt
  done
done
DS_LIB_PATH=$PWD/ab/p256a2.so timeout 900 python -m pytest tests/test_gpu_pcg.py tests/test_gpu_baseline_parity.py -q > gpurun_out/c66/tests.log 2>&1
echo "exit $?" >> gpurun_out/c66/tests.log
