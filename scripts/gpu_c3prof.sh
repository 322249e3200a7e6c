TAG=${1:-c3p}
mkdir -p gpurun_out
python -c "from paper_2305_03018_b200 import build; build.build()" > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"tonal_kernel_coop|tonal_kernel_dispatch" -s 11 -c 11 -o gpurun_out/prof_c3_$TAG \
   python scripts/run_config_once.py c3 --reps 2 > gpurun_out/ncu_c3_$TAG.log 2>&1
python scripts/ncu_summary.py gpurun_out/prof_c3_$TAG.ncu-rep gpurun_out/c3_summary_$TAG > /dev/null 2>&1
