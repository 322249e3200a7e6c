TAG=${1:-big2}
mkdir -p gpurun_out
FM_LIB=paper_2305_03018_b200/_build/ab_new.so timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_clamp.py -x -q -p no:cacheprovider > gpurun_out/tests_$TAG.log 2>&1
echo "rc=$?" >> gpurun_out/tests_$TAG.log
run() { echo "== $*" >> gpurun_out/cfg_$TAG.log; env "$@" timeout 600 python scripts/bench_configs.py --only c4,c2 --reps 30 2>&1 | grep -v "^{" >> gpurun_out/cfg_$TAG.log; }
for rep in 1 2; do
run FM_LIB=paper_2305_03018_b200/_build/ab_new.so
run FM_LIB=paper_2305_03018_b200/_build/ab_old.so
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_c4_$TAG.csv \
     python scripts/run_config_once.py c4 --reps 2 > gpurun_out/launch_c4_$TAG.log 2>&1
