# usage: bash scripts/gpu_abn.sh TAG CONFIGS name1 name2 ...  — per-config A/B of _build/ab_<name>.so libraries (2 rounds)
TAG=$1; CFGS=$2; shift 2
mkdir -p gpurun_out
for rep in 1 2; do for n in "$@"; do
  echo "== $n" >> gpurun_out/cfg_$TAG.log
  FM_LIB=paper_2305_03018_b200/_build/ab_$n.so timeout 600 python scripts/bench_configs.py --only $CFGS --modes dilate --reps 30 2>&1 | grep -v "^{" >> gpurun_out/cfg_$TAG.log
done; done
