# usage: bash scripts/gpu_ab2.sh TAG CONFIGS  — tests with ab_new.so, per-config A/B new vs old, c5 bench A/B
TAG=$1; CFGS=${2:-c1,c2,c3,c4,c5}
mkdir -p gpurun_out
FM_LIB=paper_2305_03018_b200/_build/ab_new.so timeout 1500 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/tests_$TAG.log 2>&1
echo "rc=$?" >> gpurun_out/tests_$TAG.log
run() { echo "== $*" >> gpurun_out/cfg_$TAG.log; env "$@" timeout 600 python scripts/bench_configs.py --only $CFGS --modes dilate --reps 30 2>&1 | grep -v "^{" >> gpurun_out/cfg_$TAG.log; }
for rep in 1 2; do
run FM_LIB=paper_2305_03018_b200/_build/ab_new.so
run FM_LIB=paper_2305_03018_b200/_build/ab_old.so
done
bash scripts/gpu_ab_libs.sh $TAG 2 new old
