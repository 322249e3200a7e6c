mkdir -p gpurun_out
python -c "from paper_2305_03018_b200 import build; build.build()" > gpurun_out/build_r2h.log 2>&1
timeout 900 python scripts/bench_configs.py --only c1,c2,c3,c4,c5 --reps 20 2>&1 | grep -v "^{" > gpurun_out/cfg_r2h.log
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/tests_all_r2h.log 2>&1
echo "rc=$?" >> gpurun_out/tests_all_r2h.log
