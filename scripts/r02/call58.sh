# full GPU suite + smoke on the committed state
mkdir -p gpurun_out/c58
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/c58/gpu_tests.log 2>&1
echo "exit $?" >> gpurun_out/c58/gpu_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/c58/smoke.log 2>&1
timeout 900 python -m pytest tests -m "not gpu" -q -x > gpurun_out/c58/cpu_tests.log 2>&1
echo "exit $?" >> gpurun_out/c58/cpu_tests.log
