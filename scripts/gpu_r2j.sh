mkdir -p gpurun_out
python -c "from paper_2305_03018_b200 import build; build.build()" > gpurun_out/build_r2j.log 2>&1
for v in 1 2 3 4 1 3; do echo "== FM_BIG_STEPS=$v" >> gpurun_out/cfg_r2j.log; FM_BIG_STEPS=$v timeout 600 python scripts/bench_configs.py --only c4 --modes dilate --reps 30 2>&1 | grep -v "^{" >> gpurun_out/cfg_r2j.log; done
timeout 1500 python -m pytest tests/test_gpu_reference_semantics.py tests/test_gpu_parity.py tests/test_gpu_clamp.py tests/test_gpu_strips.py -q -p no:cacheprovider > gpurun_out/tests_r2j.log 2>&1
echo "rc=$?" >> gpurun_out/tests_r2j.log
