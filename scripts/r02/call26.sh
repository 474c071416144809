for v in guard noguard; do DS_LIB_PATH=$PWD/ab/$v.so timeout 300 python bench_solver.py --nodes 16384 --reps 10 2>&1 | grep "^{" | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$v', d['nodes'], 'fw', d['forward_warp'], 'lin', d['linearize_ms'])"; done
for v in guard noguard; do DS_LIB_PATH=$PWD/ab/$v.so timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | grep "^{" | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$v', d['value'], d['e2e']['value'])"; done
