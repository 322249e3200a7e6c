mkdir -p gpurun_out
python -c "from paper_2305_03018_b200 import build; build.build()" > gpurun_out/build_r2i.log 2>&1
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/tests_all_r2i.log 2>&1
echo "rc=$?" >> gpurun_out/tests_all_r2i.log
for v in 1 0 1 0; do echo "== FM_RANGE_FLAT=$v" >> gpurun_out/cfg_r2i.log; FM_RANGE_FLAT=$v timeout 600 python scripts/bench_configs.py --only c2,c4 --modes dilate --reps 30 2>&1 | grep -v "^{" >> gpurun_out/cfg_r2i.log; done
