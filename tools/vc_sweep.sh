#!/bin/bash
# Standalone single-RHS V-cycle time vs the lanes-per-row rule (GNW_VC_T; 1000 = thread-per-row
# everywhere below 32 lanes... i.e. the old narrow kernels) at C2, C5 and C3 shapes.
mkdir -p gpurun_out
for T in ${TS:-2 3 4 6}; do
  echo "T=$T"
  GNW_VC_T=$T python tools/profile_kernels.py --config C2 --kernels vcycle --reps 20 | sed 's/^/  C2 /'
  GNW_VC_T=$T python tools/profile_kernels.py --n 1024 --m 32 --coarse-threshold 1024 --kernels vcycle --reps 10 | sed 's/^/  C5 /'
  GNW_VC_T=$T python tools/profile_kernels.py --n 2048 --m 32 --coarse-threshold 4096 --kernels vcycle --reps 10 | sed 's/^/  C3 /'
done
