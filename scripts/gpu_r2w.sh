mkdir -p gpurun_out
python -c "from paper_2305_03018_b200 import build; build.build()" > gpurun_out/build_r2w.log 2>&1
for v in 1 0 1 0; do echo "== FM_GRAPH=$v" >> gpurun_out/cfg_r2w.log; FM_GRAPH=$v timeout 900 python scripts/bench_configs.py --only c1,c2 --reps 50 2>&1 | grep -v "^{" >> gpurun_out/cfg_r2w.log; done
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/tests_all_r2w.log 2>&1
echo "rc=$?" >> gpurun_out/tests_all_r2w.log
timeout 300 python scripts/dropin_timing.py > gpurun_out/dropin_r2w.log 2>&1; timeout 300 python scripts/dropin_small.py >> gpurun_out/dropin_r2w.log 2>&1; FM_GRAPH=0 timeout 300 python scripts/dropin_small.py >> gpurun_out/dropin_r2w.log 2>&1
