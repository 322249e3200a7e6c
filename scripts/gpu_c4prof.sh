mkdir -p gpurun_out
python -c "from paper_2305_03018_b200 import build; build.build()" > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"big_|range_kernel|tonal" -s 12 -c 6 --import-source on -o gpurun_out/prof_c4 \
   python scripts/bench_configs.py --only c4 --modes dilate --reps 2 > gpurun_out/ncu_c4.log 2>&1

python scripts/ncu_summary.py gpurun_out/prof_c4.ncu-rep gpurun_out/c4_summary > /dev/null 2>&1
