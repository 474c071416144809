# The driver's round-end commands: default bench (with the CPU baseline) and the reference arm.
mkdir -p gpurun_out
( time timeout 1200 python bench.py ) > gpurun_out/bench_default.log 2>&1
echo "exit $?" >> gpurun_out/bench_default.log
( time timeout 1200 python bench.py --impl reference --steps 3 --warmup 3 ) > gpurun_out/bench_reference.log 2>&1
echo "exit $?" >> gpurun_out/bench_reference.log
nproc > gpurun_out/host_cpu.txt; lscpu | grep -E "Model name|^CPU\(s\)" >> gpurun_out/host_cpu.txt
