#!/bin/bash
# usage: bash scripts/gpu_launches.sh TAG CONFIG — per-launch duration + DRAM bytes of one config run
TAG=${1:-run}; CFG=${2:-c5}
mkdir -p gpurun_out
timeout 300 python scripts/run_config_once.py $CFG --images 3 --reps 1 > gpurun_out/once_$TAG.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size,launch__registers_per_thread --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python scripts/run_config_once.py $CFG --images 3 --reps 1 > gpurun_out/ncu_launches_$TAG.log 2>&1
echo rc=$? >> gpurun_out/ncu_launches_$TAG.log
