TAG=${1:-coop2}
mkdir -p gpurun_out
python -c "from paper_2305_03018_b200 import build; build.build()" > gpurun_out/build_$TAG.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "long_tonal or invariance or large_configs" > gpurun_out/tests_$TAG.log 2>&1
echo "rc=$?" >> gpurun_out/tests_$TAG.log
run() { echo "== $*" >> gpurun_out/cfg_$TAG.log; env "$@" timeout 600 python scripts/bench_configs.py --only c3 --modes dilate --reps 30 2>&1 | grep -v "^{" >> gpurun_out/cfg_$TAG.log; }
for rep in 1 2; do
run FM_X=0
run FM_TONAL_DISP_MAX=0
run FM_TONAL_COOP_MIN=81
run FM_TONAL_COOP_MIN=81 FM_TONAL_DISP_MAX=0
run FM_CONV_WAVES=3
run FM_CONV_WAVES=4
run FM_CONV_WAVES=6
done
