mkdir -p gpurun_out
python -c "from paper_2305_03018_b200 import build; build.build()" > gpurun_out/build_r2q.log 2>&1
timeout 300 python scripts/dropin_timing.py > gpurun_out/dropin_r2q.log 2>&1
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/tests_all_r2q.log 2>&1
echo "rc=$?" >> gpurun_out/tests_all_r2q.log
