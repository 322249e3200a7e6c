TAG=${1:-coop4}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -x -q -p no:cacheprovider > gpurun_out/tests_$TAG.log 2>&1
echo "rc=$?" >> gpurun_out/tests_$TAG.log
run() { echo "== $*" >> gpurun_out/cfg_$TAG.log; env "$@" timeout 600 python scripts/bench_configs.py --only $ONLY --modes dilate --reps 30 2>&1 | grep -v "^{" >> gpurun_out/cfg_$TAG.log; }
for rep in 1 2; do
ONLY=c3,c2,c4
run FM_LIB=paper_2305_03018_b200/_build/ab_magic.so
run FM_LIB=paper_2305_03018_b200/_build/ab_cvt.so
done
bash scripts/gpu_ab_libs.sh $TAG 3 magic cvt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_c3_$TAG.csv \
     python scripts/run_config_once.py c3 --reps 2 > gpurun_out/launch_c3_$TAG.log 2>&1
