#!/bin/bash
# usage: bash scripts/gpu_profile.sh TAG  -> full bench line, one-step launch list with DRAM bytes,
# and one ncu --set full capture of the conv / dominant tonal / range kernels (4-image launch)
TAG=${1:-run}
mkdir -p gpurun_out
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_full_$TAG.log 2>&1; echo bench_rc=$? >> gpurun_out/bench_full_$TAG.log
timeout 600 python bench.py --profile-step --no-cpu-baseline > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   --log-file gpurun_out/launches_$TAG.csv python bench.py --profile-step --no-cpu-baseline > gpurun_out/ncu_launches_$TAG.log 2>&1
echo launches_rc=$? >> gpurun_out/ncu_launches_$TAG.log
timeout 300 python bench.py --images 4 --profile-step --no-cpu-baseline > gpurun_out/bench_small_$TAG.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:"tile128_kernelIhLb0E|tonal_kernel_pipeILi18E|range_kernelILi0E" -c 3 -o gpurun_out/prof_$TAG \
   python bench.py --images 4 --profile-step --no-cpu-baseline > gpurun_out/ncu_$TAG.log 2>&1
echo ncu_rc=$? >> gpurun_out/ncu_$TAG.log
