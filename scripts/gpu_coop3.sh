TAG=${1:-coop3}
mkdir -p gpurun_out
python -c "from paper_2305_03018_b200 import build; build.build()" > gpurun_out/build_$TAG.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "long_tonal or invariance or large_configs" > gpurun_out/tests_$TAG.log 2>&1
echo "rc=$?" >> gpurun_out/tests_$TAG.log
run() { echo "== $*" >> gpurun_out/cfg_$TAG.log; env "$@" timeout 600 python scripts/bench_configs.py --only $ONLY --modes dilate --reps 30 2>&1 | grep -v "^{" >> gpurun_out/cfg_$TAG.log; }
for rep in 1 2; do
ONLY=c3
run FM_X=0
run FM_TONAL_DISP_MAX=0
run FM_TONAL_COOP_MIN=81
ONLY=c1,c2
run FM_CONV_WAVES=2
run FM_CONV_WAVES=4
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_c3_$TAG.csv \
     python scripts/run_config_once.py c3 --reps 2 > gpurun_out/launch_c3_$TAG.log 2>&1
