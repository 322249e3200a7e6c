TAG=${1:-coop}
mkdir -p gpurun_out
python -c "from paper_2305_03018_b200 import build; build.build()" > gpurun_out/build_$TAG.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "long_tonal or invariance or large_configs" > gpurun_out/tests_$TAG.log 2>&1
echo "rc=$?" >> gpurun_out/tests_$TAG.log
for v in 1 0 1 0; do echo "== FM_TONAL_COOP=$v" >> gpurun_out/cfg_$TAG.log; FM_TONAL_COOP=$v timeout 600 python scripts/bench_configs.py --only c3 --reps 20 2>&1 | grep -v "^{" >> gpurun_out/cfg_$TAG.log; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_c3_$TAG.csv \
     python scripts/run_config_once.py c3 --reps 2 > gpurun_out/launch_c3_$TAG.log 2>&1
