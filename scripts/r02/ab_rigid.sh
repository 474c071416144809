for i in 1 2; do
DS_RIGID_GRID=296 timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline 2>&1 | grep "^{" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cap296', d['value'], d['e2e']['value'], d['kernels']['rigid_icp'])"
timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline 2>&1 | grep "^{" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('nocap', d['value'], d['e2e']['value'], d['kernels']['rigid_icp'])"
done
