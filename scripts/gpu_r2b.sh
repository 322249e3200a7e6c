mkdir -p gpurun_out
python -c "from paper_2305_03018_b200 import build; build.build()" > gpurun_out/build_r2b.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_fft_conv.py tests/test_gpu_strips.py -q -p no:cacheprovider > gpurun_out/tests_new_r2b.log 2>&1
echo "rc=$?" >> gpurun_out/tests_new_r2b.log
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/tests_all_r2b.log 2>&1
echo "rc=$?" >> gpurun_out/tests_all_r2b.log
for c in c3 c4; do timeout 600 python bench.py --config $c --no-cpu-baseline --steps 10 > gpurun_out/bench_${c}_r2b.log 2>&1; echo "rc=$?" >> gpurun_out/bench_${c}_r2b.log; done
