# final numbers on the committed build
mkdir -p gpurun_out/c74
timeout 1200 python bench.py > gpurun_out/c74/bench_default.json 2> gpurun_out/c74/bench_default.err
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/c74/bench_20.json 2> gpurun_out/c74/bench_20.err
timeout 900 python bench.py --config cfg3 --no-cpu-baseline > gpurun_out/c74/bench_cfg3.json 2>&1
timeout 900 python bench.py --config cfg1 > gpurun_out/c74/bench_cfg1.json 2>&1
timeout 900 python bench.py --sequences 8 --steps 40 --no-cpu-baseline > gpurun_out/c74/bench_cfg5.json 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/c74/smoke.log 2>&1
