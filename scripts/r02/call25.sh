timeout 300 python -m pytest tests/test_gpu_pcg.py -q -k spmv > gpurun_out/r02_c25_test.log 2>&1
timeout 600 python bench_solver.py --nodes 4096 16384 --reps 10 > gpurun_out/r02_c25_tma.log 2>&1
DS_SPMV_TMA=0 timeout 600 python bench_solver.py --nodes 4096 16384 --reps 10 > gpurun_out/r02_c25_rows.log 2>&1
