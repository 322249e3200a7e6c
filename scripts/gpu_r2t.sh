mkdir -p gpurun_out
python -c "from paper_2305_03018_b200 import build; build.build()" > gpurun_out/build_r2t.log 2>&1
timeout 900 python scripts/bench_configs.py --reps 20 --images 8 2>&1 | grep -v "^{" > gpurun_out/cfg_r2t.log
FM_CHAT16=0 timeout 900 python scripts/bench_configs.py --only c3 --reps 20 2>&1 | grep -v "^{" >> gpurun_out/cfg_r2t.log
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/tests_all_r2t.log 2>&1
echo "rc=$?" >> gpurun_out/tests_all_r2t.log
