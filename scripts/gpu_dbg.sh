mkdir -p gpurun_out
python -c "from paper_2305_03018_b200 import build; build.build()" > gpurun_out/build_dbg.log 2>&1
FM_PLAN_DEBUG=1 timeout 600 python scripts/bench_configs.py --only c1 --modes dilate --reps 50 > gpurun_out/dbg3.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size,launch__registers_per_thread --csv python scripts/bench_configs.py --only c1 --modes dilate --reps 2 > gpurun_out/dbg3_ncu.csv 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "ladder or invariance" > gpurun_out/dbg3_tests.log 2>&1
