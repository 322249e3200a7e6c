mkdir -p gpurun_out
python -c "from paper_2305_03018_b200 import build; build.build()" > gpurun_out/build_r2m.log 2>&1
for v in 0 48 24 96 0 48; do echo "== FM_BIG_L2_MB=$v" >> gpurun_out/cfg_r2m.log; FM_BIG_L2_MB=$v timeout 600 python scripts/bench_configs.py --only c4 --modes dilate --reps 30 2>&1 | grep -v "^{" >> gpurun_out/cfg_r2m.log; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_envelope.py tests/test_gpu_strips.py -q -p no:cacheprovider > gpurun_out/tests_r2m.log 2>&1
echo "rc=$?" >> gpurun_out/tests_r2m.log
