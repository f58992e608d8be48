#!/bin/bash
# Woodbury setup kernels: plain timings, launch list, and --set full of the first K kernels.
#   bash tools/ncu_setup.sh <tag> <n> <m> <coarse_threshold> [K]
tag=${1:-c2}; n=${2:-512}; m=${3:-256}; ct=${4:-64}; K=${5:-6}
mkdir -p gpurun_out
python tools/profile_setup.py --n $n --m $m --coarse-threshold $ct > gpurun_out/setup_${tag}_plain.txt 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --profile-from-start off --csv --log-file gpurun_out/setup_${tag}_launches.csv \
    python tools/profile_setup.py --n $n --m $m --coarse-threshold $ct > gpurun_out/setup_${tag}_ncu.log 2>&1
ncu --set full --clock-control none --import-source on --profile-from-start off -c $K \
    -o gpurun_out/setup_${tag}_full -f \
    python tools/profile_setup.py --n $n --m $m --coarse-threshold $ct > gpurun_out/setup_${tag}_full.log 2>&1
