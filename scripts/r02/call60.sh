# config 3 / 5 bench lines on the final build (no DS_HOST_LM leak)
mkdir -p gpurun_out/c60
unset DS_HOST_LM
timeout 900 python bench.py --config cfg3 --no-cpu-baseline > gpurun_out/c60/bench_cfg3.json 2>&1
timeout 900 python bench.py --sequences 8 --steps 40 --no-cpu-baseline > gpurun_out/c60/bench_cfg5.json 2>&1
