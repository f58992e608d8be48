#!/bin/bash
# One measurement pass on the GPU box: bench lines for every config, the launch list of the bench
# command's timed region (GNW_NO_GRAPH: ncu does not list kernels inside conditional graph
# bodies), a launch list of one C2 solve, and ncu --set full of the C2 per-iteration kernels and
# the capacitance GEMM.  Outputs under gpurun_out/.
mkdir -p gpurun_out
for c in ${CONFIGS:-C2 C1 C4 C5 C3}; do
  timeout 1500 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  echo "$c rc=$?"
done
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference_arm.json 2> gpurun_out/bench_reference_arm.err
echo "reference arm rc=$?"
GNW_NO_GRAPH=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --profile-from-start off --csv --log-file gpurun_out/bench_c2_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2_ncu.log 2>&1
echo "bench launches rc=$?"
GNW_NO_GRAPH=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --profile-from-start off --csv --log-file gpurun_out/solve_c2_launches.csv python tools/profile_one.py > gpurun_out/solve_c2_ncu.log 2>&1
echo "launches rc=$?"
ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:"k_row_gemv|k_saddle|k_col_sweep|k_finish_prec|k_minres_update|k_vcl_up|k_vcl_restrict|k_coarse_inverse1|k_combine_elem" -c 16 \
  -o gpurun_out/iter_c2_full -f python tools/profile_kernels.py --config C2 --kernels row_gemv,saddle_fused,col_sweep,finish_lean,vcycle,update,combine_prec --reps 1 > gpurun_out/iter_c2_full.log 2>&1
echo "full rc=$?"
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"k_dgemm_tma|k_mvcf_up_rows" -c 2 \
  -o gpurun_out/setup_c2_full -f python tools/profile_setup.py --n 512 --m 256 > gpurun_out/setup_c2_full.log 2>&1
echo "setup full rc=$?"
