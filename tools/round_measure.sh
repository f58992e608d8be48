#!/bin/bash
# One measurement pass on the GPU box: bench lines for every config, a launch list of one C2
# solve, and ncu --set full of the C2 per-iteration kernels.  Outputs under gpurun_out/.
mkdir -p gpurun_out
for c in ${CONFIGS:-C2 C1 C4 C5 C3}; do
  timeout 1500 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  echo "$c rc=$?"
done
GNW_NO_GRAPH=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --profile-from-start off --csv --log-file gpurun_out/solve_c2_launches.csv python tools/profile_one.py > gpurun_out/solve_c2_ncu.log 2>&1
echo "launches rc=$?"
ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:"k_row_gemv|k_saddle|k_col_sweep|k_finish_prec|k_minres_update|k_vcs_down|k_vcs_up2|k_vcg_down" -c 10 \
  -o gpurun_out/iter_c2_full -f python tools/profile_kernels.py --config C2 --kernels row_gemv,saddle_fused,col_sweep,finish_lean,vcycle,update --reps 1 > gpurun_out/iter_c2_full.log 2>&1
echo "full rc=$?"
