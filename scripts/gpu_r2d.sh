mkdir -p gpurun_out
python -c "from paper_2305_03018_b200 import build; build.build()" > gpurun_out/build_r2d.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_envelope.py -q -p no:cacheprovider > gpurun_out/tests_env_r2d.log 2>&1
echo "rc=$?" >> gpurun_out/tests_env_r2d.log
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/tests_all_r2d.log 2>&1
echo "rc=$?" >> gpurun_out/tests_all_r2d.log
