# launch list of one config: bash scripts/gpu_ll1.sh CFG TAG
C=$1; TAG=$2
mkdir -p gpurun_out
python -c "from paper_2305_03018_b200 import build; build.build()" > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_${C}_$TAG.csv \
     python scripts/run_config_once.py $C --reps 2 > gpurun_out/launch_${C}_$TAG.log 2>&1
