TAG=${1:-rng}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/tests_$TAG.log 2>&1
echo "rc=$?" >> gpurun_out/tests_$TAG.log
run() { echo "== $*" >> gpurun_out/cfg_$TAG.log; env "$@" timeout 600 python scripts/bench_configs.py --only c2,c3,c4,c5 --modes dilate --reps 30 2>&1 | grep -v "^{" >> gpurun_out/cfg_$TAG.log; }
for rep in 1 2; do
run FM_X=0
run FM_RANGE_ALIGNED=0
done
bash scripts/gpu_benchab.sh $TAG - FM_RANGE_ALIGNED=0 - FM_RANGE_ALIGNED=0
