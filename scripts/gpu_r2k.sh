mkdir -p gpurun_out
python -c "from paper_2305_03018_b200 import build; build.build()" > gpurun_out/build_r2k.log 2>&1
timeout 600 python scripts/probe_spec.py > gpurun_out/probe_r2k.log 2>&1
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/tests_all_r2k.log 2>&1
echo "rc=$?" >> gpurun_out/tests_all_r2k.log
timeout 600 python scripts/bench_configs.py --only c1,c2 --reps 50 2>&1 | grep -v "^{" > gpurun_out/cfg_r2k.log
