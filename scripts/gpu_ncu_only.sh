TAG=$1
timeout 300 python bench.py --images 4 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/bench_small_$TAG.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:"tile128_kernelIhLb0E|tonal_kernel_pipeILi18E|range_kernelILi0E" -s 3 -c 3 -o gpurun_out/prof_$TAG \
   python bench.py --images 4 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_$TAG.log 2>&1
echo ncu_rc=$? >> gpurun_out/ncu_$TAG.log
