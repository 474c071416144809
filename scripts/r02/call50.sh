# PCG: pipelined loop's CTA reductions on dedicated buffers (two barriers fewer per iteration)
mkdir -p gpurun_out/c50
timeout 900 python -m pytest tests/test_gpu_pcg.py tests/test_gpu_solve_fusion.py -q -x > gpurun_out/c50/tests.log 2>&1
echo "tests exit $?" >> gpurun_out/c50/tests.log
bash scripts/gpu_ab_libs.sh base cur
cp gpurun_out/ab_summary.txt gpurun_out/c50/ab.txt
