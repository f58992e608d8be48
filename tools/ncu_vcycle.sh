#!/bin/bash
# V-cycle kernels at large shapes: launch list (time + DRAM bytes) and one --set full capture.
#   bash tools/ncu_vcycle.sh <tag> <n> <coarse_threshold>
tag=${1:-c3}; n=${2:-2048}; ct=${3:-4096}
mkdir -p gpurun_out
python tools/profile_kernels.py --n $n --m 32 --coarse-threshold $ct --kernels vcycle --reps 5 > gpurun_out/vc_${tag}_plain.txt 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size,sm__warps_active.avg.pct_of_peak_sustained_active \
    --clock-control none --profile-from-start off --csv --log-file gpurun_out/vc_${tag}_launches.csv \
    python tools/profile_kernels.py --n $n --m 32 --coarse-threshold $ct --kernels vcycle --reps 1 > gpurun_out/vc_${tag}_ncu.log 2>&1
ncu --set full --clock-control none --import-source on --profile-from-start off -c 8 \
    -o gpurun_out/vc_${tag}_full -f \
    python tools/profile_kernels.py --n $n --m 32 --coarse-threshold $ct --kernels vcycle --reps 1 > gpurun_out/vc_${tag}_full.log 2>&1
