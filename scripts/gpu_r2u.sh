mkdir -p gpurun_out
python -c "from paper_2305_03018_b200 import build; build.build()" > gpurun_out/build_r2u.log 2>&1
for v in 40 80 40 80; do echo "== FM_TONAL_PIPE_MAX=$v" >> gpurun_out/cfg_r2u.log; FM_TONAL_PIPE_MAX=$v timeout 900 python scripts/bench_configs.py --only c3,c5 --modes dilate --reps 20 --images 8 2>&1 | grep -v "^{" >> gpurun_out/cfg_r2u.log; done
