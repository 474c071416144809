python -m pytest tests/test_gpu_solve_fusion.py -m gpu -x -q -k "incremental or grid_knn or sequence" 2>&1 | tail -3
