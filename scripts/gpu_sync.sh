TAG=${1:-sync}
mkdir -p gpurun_out
run() { echo "== $*" >> gpurun_out/cfg_$TAG.log; env "$@" timeout 600 python scripts/bench_configs.py --only c2,c4 --modes dilate --reps 30 2>&1 | grep -v "^{" >> gpurun_out/cfg_$TAG.log; }
for rep in 1 2; do
run FM_X=0
run FM_RANGE_SYNC=1
run FM_RANGE_TAPS=32
run FM_RANGE_TAPS=64
done
