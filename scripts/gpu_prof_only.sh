TAG=r2b
mkdir -p gpurun_out
python -c "from paper_2305_03018_b200 import build; build.build()" > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:"tile128_kernelIhLb0E|tonal_kernel_pipeILi18E|range_kernelILi0E" -c 3 -o gpurun_out/prof_$TAG \
   python bench.py --images 4 --profile-step --no-cpu-baseline > gpurun_out/ncu_$TAG.log 2>&1
echo ncu_rc=$? >> gpurun_out/ncu_$TAG.log
