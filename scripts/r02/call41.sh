timeout 900 python -m pytest tests/test_gpu_solve_fusion.py tests/test_gpu_baseline_parity.py tests/test_gpu_acceptance.py -q -x > gpurun_out/r02_c41_tests.log 2>&1
bash scripts/gpu_ab_libs.sh base3 energy
