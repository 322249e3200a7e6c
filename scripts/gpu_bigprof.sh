TAG=${1:-bp}
mkdir -p gpurun_out
python -c "from paper_2305_03018_b200 import build; build.build()" > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base mangled -k regex:"big_rows_kernelILb1ELb0E|big_cols_kernelILb0E|big_rows_kernelILb0ELb0E" -s 3 -c 3 -o gpurun_out/prof_big_$TAG \
   python scripts/run_config_once.py c4 --reps 3 > gpurun_out/ncu_big_$TAG.log 2>&1
ncu -i gpurun_out/prof_big_$TAG.ncu-rep --page source --csv > gpurun_out/big_source_$TAG.csv 2>/dev/null
python scripts/ncu_summary.py gpurun_out/prof_big_$TAG.ncu-rep gpurun_out/big_summary_$TAG > /dev/null 2>&1
