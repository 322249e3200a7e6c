TAG=${1:-small}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/tests_$TAG.log 2>&1
echo "rc=$?" >> gpurun_out/tests_$TAG.log
run() { echo "== $*" >> gpurun_out/cfg_$TAG.log; env "$@" timeout 600 python scripts/bench_configs.py --only c1,c2 --modes dilate --reps 100 2>&1 | grep -v "^{" >> gpurun_out/cfg_$TAG.log; }
for rep in 1 2 3; do
run FM_LIB=paper_2305_03018_b200/_build/ab_new.so
run FM_LIB=paper_2305_03018_b200/_build/ab_old.so
done
