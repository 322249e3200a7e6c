mkdir -p gpurun_out
python -c "from paper_2305_03018_b200 import build; build.build()" > gpurun_out/build_r2v.log 2>&1
timeout 900 python scripts/bench_configs.py --only c2,c4,c5,c3 --modes dilate --reps 20 --images 8 2>&1 | grep -v "^{" > gpurun_out/cfg_r2v.log
timeout 900 python -m pytest tests/test_gpu_clamp.py tests/test_gpu_parity.py tests/test_gpu_fuzz.py -q -p no:cacheprovider > gpurun_out/tests_r2v.log 2>&1
echo "rc=$?" >> gpurun_out/tests_r2v.log
