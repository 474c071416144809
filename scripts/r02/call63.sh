# PCG CTA size A/B (512 / 384 / 256 threads)
mkdir -p gpurun_out/c63
for v in p256 p384; do
  DS_LIB_PATH=$PWD/ab/$v.so timeout 600 python -m pytest tests/test_gpu_pcg.py tests/test_gpu_solve_fusion.py -q -x > gpurun_out/c63/tests_$v.log 2>&1
  echo "exit $?" >> gpurun_out/c63/tests_$v.log
done
: > gpurun_out/c63/ab.txt
for r in 1 2; do
  for v in p512 p384 p256; do
    DS_LIB_PATH=$PWD/ab/$v.so timeout 900 python bench.py --no-cpu-baseline --steps 60 > gpurun_out/c63/run.log 2>&1
    echo "$v run$r $(grep '^{' gpurun_out/c63/run.log | cut -c30-60) $(grep '^{' gpurun_out/c63/run.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["kernels"]["pcg"]["mean_launch_us"])')" >> gpurun_out/c63/ab.txt
  done
done
