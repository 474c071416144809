mkdir -p gpurun_out/c67
: > gpurun_out/c67/ab.txt
for r in 1 2; do
  for v in c64 c128; do
    DS_LIB_PATH=$PWD/ab/$v.so timeout 900 python bench.py --no-cpu-baseline --steps 60 > gpurun_out/c67/run.log 2>&1
    echo "$v run$r $(grep '^{' gpurun_out/c67/run.log | cut -c30-60) $(grep '^{' gpurun_out/c67/run.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); k=d["kernels"]; print(k["block_assembly"]["mean_launch_us"], k["reduce"]["mean_launch_us"])')" >> gpurun_out/c67/ab.txt
  done
done
