# the compiled reference (oracle/_ref) on the GPU box: device-vs-reference tests, the reference arm
mkdir -p gpurun_out/c51
timeout 900 python -m pytest tests/test_gpu_baseline_parity.py -q -k "compiled_reference" > gpurun_out/c51/tests_gpu.log 2>&1
echo "exit $?" >> gpurun_out/c51/tests_gpu.log
timeout 900 python -m pytest tests/test_ref_oracle.py -q > gpurun_out/c51/tests_ref.log 2>&1
echo "exit $?" >> gpurun_out/c51/tests_ref.log
timeout 900 python bench.py --impl reference > gpurun_out/c51/ref_cfg2.json 2> gpurun_out/c51/ref_cfg2.err
timeout 600 python bench.py --impl reference --config cfg1 > gpurun_out/c51/ref_cfg1.json 2> gpurun_out/c51/ref_cfg1.err
