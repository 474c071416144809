mkdir -p gpurun_out
./scripts/microbench/gjbench_nofma > gpurun_out/gjbench.log 2>&1
./scripts/microbench/gjbench_rcp >> gpurun_out/gjbench.log 2>&1
