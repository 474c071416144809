# final numbers on the committed build
mkdir -p gpurun_out/c68
timeout 1200 python bench.py > gpurun_out/c68/bench_default.json 2> gpurun_out/c68/bench_default.err
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/c68/bench_20.json 2> gpurun_out/c68/bench_20.err
timeout 900 python bench.py --impl reference > gpurun_out/c68/ref_cfg2.json 2> gpurun_out/c68/ref_cfg2.err
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/c68/smoke.log 2>&1
