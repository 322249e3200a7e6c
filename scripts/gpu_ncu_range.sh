#!/bin/bash
TAG=${1:-run}
mkdir -p gpurun_out
for c in c2 c4; do
  timeout 300 python scripts/run_config_once.py $c > gpurun_out/once_${c}_$TAG.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:range_kernel -s 1 -c 1 -o gpurun_out/range_${c}_$TAG python scripts/run_config_once.py $c > gpurun_out/ncu_range_${c}_$TAG.log 2>&1
  echo rc=$? >> gpurun_out/ncu_range_${c}_$TAG.log
done
