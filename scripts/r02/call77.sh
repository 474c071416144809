# k_energy: 1 / 2 / 4 pixels per thread packed per CTA
mkdir -p gpurun_out/c77
for v in e2 e4; do
  DS_LIB_PATH=$PWD/ab/$v.so timeout 900 python -m pytest tests/test_gpu_solve_fusion.py tests/test_gpu_baseline_parity.py -q -x > gpurun_out/c77/tests_$v.log 2>&1
  echo "exit $?" >> gpurun_out/c77/tests_$v.log
done
: > gpurun_out/c77/ab.txt
for r in 1 2; do
  for v in e1 e2 e4; do
    DS_LIB_PATH=$PWD/ab/$v.so timeout 900 python bench.py --no-cpu-baseline --steps 60 > gpurun_out/c77/run.log 2>&1
    echo "$v run$r $(grep '^{' gpurun_out/c77/run.log | cut -c30-60) $(grep '^{' gpurun_out/c77/run.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["kernels"]["energy"]["mean_launch_us"])')" >> gpurun_out/c77/ab.txt
  done
done
