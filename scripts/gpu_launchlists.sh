# launch lists (ncu gpu__time_duration) of the single-image configs: bash scripts/gpu_launchlists.sh TAG
TAG=${1:-ll}
mkdir -p gpurun_out
python -c "from paper_2305_03018_b200 import build; build.build()" > /dev/null 2>&1
for c in c1 c2 c3 c4; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_${c}_$TAG.csv \
     python scripts/run_config_once.py $c --reps 2 > gpurun_out/launch_${c}_$TAG.log 2>&1
done
