TAG=${1:-coop5}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_strips.py tests/test_gpu_envelope.py -x -q -p no:cacheprovider > gpurun_out/tests_$TAG.log 2>&1
echo "rc=$?" >> gpurun_out/tests_$TAG.log
run() { echo "== $*" >> gpurun_out/cfg_$TAG.log; env "$@" timeout 600 python scripts/bench_configs.py --only c3 --reps 30 2>&1 | grep -v "^{" >> gpurun_out/cfg_$TAG.log; }
for rep in 1 2; do
run FM_X=0
run FM_Y=0
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_c3_$TAG.csv \
     python scripts/run_config_once.py c3 --reps 2 > gpurun_out/launch_c3_$TAG.log 2>&1
