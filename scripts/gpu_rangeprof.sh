mkdir -p gpurun_out
python -c "from paper_2305_03018_b200 import build; build.build()" > /dev/null 2>&1
for c in c2 c4; do
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"range_kernel" -s 3 -c 1 -o /tmp/prof_range_$c \
   python scripts/bench_configs.py --only $c --modes dilate --reps 3 > gpurun_out/ncu_range_$c.log 2>&1
ncu -i /tmp/prof_range_$c.ncu-rep --page source --csv --print-source sass > gpurun_out/range_src_$c.csv 2>&1
ncu -i /tmp/prof_range_$c.ncu-rep --page raw --csv > gpurun_out/range_raw_$c.csv 2>&1
done
