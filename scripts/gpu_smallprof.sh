TAG=${1:-sp}
mkdir -p gpurun_out
python -c "from paper_2305_03018_b200 import build; build.build()" > /dev/null 2>&1
for c in c1 c2; do
FM_GRAPH=0 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"range_kernel|tile_conv|tonal" -s 6 -c 3 -o gpurun_out/prof_${c}_$TAG \
   python scripts/run_config_once.py $c --reps 3 > gpurun_out/ncu_${c}_$TAG.log 2>&1
python scripts/ncu_summary.py gpurun_out/prof_${c}_$TAG.ncu-rep gpurun_out/${c}_summary_$TAG > /dev/null 2>&1
done
