mkdir -p gpurun_out
python -c "from paper_2305_03018_b200 import build; build.build()" > gpurun_out/build_r2e.log 2>&1
for v in 1 0 1 0; do echo "== FM_DEVDISPATCH=$v" >> gpurun_out/cfg_r2e.log; FM_DEVDISPATCH=$v timeout 600 python scripts/bench_configs.py --only c1,c2,c4 --modes dilate --reps 50 2>&1 | grep -v "^{" >> gpurun_out/cfg_r2e.log; done
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/tests_all_r2e.log 2>&1
echo "rc=$?" >> gpurun_out/tests_all_r2e.log
