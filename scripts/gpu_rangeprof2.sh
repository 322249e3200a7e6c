TAG=${1:-rp}
mkdir -p gpurun_out
python -c "from paper_2305_03018_b200 import build; build.build()" > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"range_kernel" -s 3 -c 1 -o gpurun_out/prof_range_$TAG \
   python scripts/run_config_once.py c4 --reps 4 > gpurun_out/ncu_range_$TAG.log 2>&1
ncu -i gpurun_out/prof_range_$TAG.ncu-rep --page source --csv > gpurun_out/range_source_$TAG.csv 2>/dev/null
python scripts/ncu_summary.py gpurun_out/prof_range_$TAG.ncu-rep gpurun_out/range_summary_$TAG > /dev/null 2>&1
