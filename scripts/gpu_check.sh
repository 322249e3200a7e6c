#!/bin/bash
# usage: bash scripts/gpu_check.sh TAG [ncu]
TAG=${1:-run}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -s -x > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu_$TAG.log
timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bench_$TAG.log 2>&1; echo bench_rc=$? >> gpurun_out/bench_$TAG.log
if [ "$2" == "ncu" ]; then
  timeout 300 python bench.py --images 4 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/bench_small_$TAG.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:"ILi128ELi128ELi512ELb1ELb0E|tonal_kernel_tILi30E" -s 2 -c 2 -o gpurun_out/prof_$TAG python bench.py --images 4 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_$TAG.log 2>&1
  echo ncu_rc=$? >> gpurun_out/ncu_$TAG.log
fi
