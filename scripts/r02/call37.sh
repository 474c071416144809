for m in 2 0 2 0; do DS_SPMV_TMA=$m timeout 300 python bench_solver.py --nodes 4096 16384 --reps 10 2>&1 | grep "^{" | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('mode $m', d['nodes'], d['spmv'])"; done
DS_SPMV_TMA=2 timeout 300 python -m pytest tests/test_gpu_pcg.py -q -k spmv 2>&1 | tail -1
DS_SPMV_TMA=2 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:k_bsr_spmv -c 2 python bench_solver.py --nodes 16384 --reps 2 2>&1 | grep -E "k_bsr|duration|bytes_read|throughput"
DS_SPMV_TMA=0 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:k_bsr_spmv -c 2 python bench_solver.py --nodes 16384 --reps 2 2>&1 | grep -E "k_bsr|duration|bytes_read|throughput"
