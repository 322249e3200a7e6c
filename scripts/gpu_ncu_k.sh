#!/bin/bash
# usage: bash scripts/gpu_ncu_k.sh TAG CONFIG REGEX [COUNT] — ncu --set full of matching kernels in one config run
TAG=${1:-run}; CFG=${2:-c5}; RX=${3:-tonal}; CNT=${4:-1}
mkdir -p gpurun_out
timeout 300 python scripts/run_config_once.py $CFG --images 3 --reps 1 > gpurun_out/once_$TAG.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:"$RX" -c $CNT -o gpurun_out/k_$TAG python scripts/run_config_once.py $CFG --images 3 --reps 1 > gpurun_out/ncu_k_$TAG.log 2>&1
echo rc=$? >> gpurun_out/ncu_k_$TAG.log
