mkdir -p gpurun_out/c65
: > gpurun_out/c65/ab.txt
for r in 1 2; do
  for v in p256a p128a; do
    DS_LIB_PATH=$PWD/ab/$v.so timeout 900 python bench.py --no-cpu-baseline --steps 60 > gpurun_out/c65/run.log 2>&1
    echo "$v run$r $(grep '^{' gpurun_out/c65/run.log | cut -c30-60) $(grep '^{' gpurun_out/c65/run.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["kernels"]["pcg"]["mean_launch_us"])')" >> gpurun_out/c65/ab.txt
  done
done
DS_LIB_PATH=$PWD/ab/p128a.so timeout 900 python -m pytest tests/test_gpu_pcg.py tests/test_gpu_baseline_parity.py -q > gpurun_out/c65/tests.log 2>&1
echo "exit $?" >> gpurun_out/c65/tests.log
