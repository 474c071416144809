# k_assoc_pair_terms: 1 / 2 / 4 pixels per thread (with k_energy at 2)
mkdir -p gpurun_out/c78
for v in p2e2 p4e2; do
  DS_LIB_PATH=$PWD/ab/$v.so timeout 900 python -m pytest tests/test_gpu_stages.py tests/test_gpu_baseline_parity.py -q -x > gpurun_out/c78/tests_$v.log 2>&1
  echo "exit $?" >> gpurun_out/c78/tests_$v.log
done
: > gpurun_out/c78/ab.txt
for r in 1 2; do
  for v in p1e2 p2e2 p4e2; do
    DS_LIB_PATH=$PWD/ab/$v.so timeout 900 python bench.py --no-cpu-baseline --steps 60 > gpurun_out/c78/run.log 2>&1
    echo "$v run$r $(grep '^{' gpurun_out/c78/run.log | cut -c30-60) $(grep '^{' gpurun_out/c78/run.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["kernels"]["pair_terms"]["mean_launch_us"])')" >> gpurun_out/c78/ab.txt
  done
done
