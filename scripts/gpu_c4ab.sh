TAG=${1:-c4ab}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_envelope.py tests/test_gpu_strips.py tests/test_gpu_fft_conv.py -x -q -p no:cacheprovider > gpurun_out/tests_$TAG.log 2>&1
echo "rc=$?" >> gpurun_out/tests_$TAG.log
run() { echo "== $*" >> gpurun_out/cfg_$TAG.log; env "$@" timeout 600 python scripts/bench_configs.py --only c4 --reps 30 2>&1 | grep -v "^{" >> gpurun_out/cfg_$TAG.log; }
for rep in 1 2; do
run FM_X=0
run FM_BIG_PAIR=0
run FM_TONAL_PIPE_MIN=0
run FM_TONAL_PIPE_MIN=5
done
