# Round-2 profile set: plain run first, then ncu (launch list + full sets).
mkdir -p gpurun_out/prof_final
CMD2="python scripts/profile_frames.py 20 2"
export DS_HOST_LM=1   # per-kernel launches (the device LM graph hides kernels from ncu); unset before any bench line
$CMD2 > gpurun_out/prof_final/plain_cfg2.log 2>&1 || exit 1
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/prof_final/launches_cfg2.csv $CMD2 > gpurun_out/prof_final/ncu_launches.log 2>&1
for k in k_energy k_assemble_chunks k_pcg k_assoc_pair_terms k_model_splat; do
  timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on \
      -k regex:"^$k" -s 2 -c 1 -o gpurun_out/prof_final/cfg2_$k -f $CMD2 > gpurun_out/prof_final/ncu_cfg2_$k.log 2>&1
done
# refresh the other configs' bench lines on the final build (device LM graph)
unset DS_HOST_LM
timeout 900 python bench.py --config cfg3 --no-cpu-baseline > gpurun_out/prof_final/bench_cfg3.json 2>&1
timeout 900 python bench.py --sequences 8 --steps 40 --no-cpu-baseline > gpurun_out/prof_final/bench_cfg5.json 2>&1
timeout 900 python bench.py --config cfg1 > gpurun_out/prof_final/bench_cfg1.json 2>&1
timeout 900 python bench_solver.py > gpurun_out/prof_final/bench_solver.json 2>&1
