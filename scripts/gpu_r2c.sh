mkdir -p gpurun_out
python -c "from paper_2305_03018_b200 import build; build.build()" > gpurun_out/build_r2c.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_fft_conv.py tests/test_gpu_frontend.py -q -p no:cacheprovider > gpurun_out/tests_new_r2c.log 2>&1
echo "rc=$?" >> gpurun_out/tests_new_r2c.log
