mkdir -p gpurun_out
python -c "from paper_2305_03018_b200 import build; build.build()" > gpurun_out/build_r2f.log 2>&1
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/tests_all_r2f.log 2>&1
echo "rc=$?" >> gpurun_out/tests_all_r2f.log
timeout 600 python scripts/bench_configs.py --only c1,c2,c4 --modes dilate --reps 50 2>&1 | grep -v "^{" > gpurun_out/cfg_r2f.log
for c in c1 c2 c4; do
timeout 600 ncu --set full --clock-control none --import-source on -s 20 -c 6 -o gpurun_out/prof_r2f_$c \
   python scripts/bench_configs.py --only $c --modes dilate --reps 3 > gpurun_out/ncu_r2f_$c.log 2>&1
done
