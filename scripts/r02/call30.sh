for v in noguard guard5; do
DS_LIB_PATH=$PWD/ab/$v.so timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,smsp__sass_inst_executed_op_local_ld.sum,smsp__sass_inst_executed_op_local_st.sum,smsp__inst_executed_pipe_fp64.sum --clock-control none -k regex:k_forward_warp -c 3 python bench_solver.py --nodes 16384 --reps 3 > gpurun_out/r02_c30_$v.log 2>&1
done
