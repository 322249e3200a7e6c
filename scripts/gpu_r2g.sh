mkdir -p gpurun_out
python -c "from paper_2305_03018_b200 import build; build.build()" > gpurun_out/build_r2g.log 2>&1
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/tests_all_r2g.log 2>&1
echo "rc=$?" >> gpurun_out/tests_all_r2g.log
FM_FUSE=1 timeout 900 python -m pytest tests/test_gpu_bench_parity.py tests/test_gpu_parity.py tests/test_gpu_fuzz.py -q -p no:cacheprovider > gpurun_out/tests_fused_r2g.log 2>&1
echo "rc=$?" >> gpurun_out/tests_fused_r2g.log
timeout 600 python scripts/bench_configs.py --only c1,c2,c4 --modes dilate --reps 50 2>&1 | grep -v "^{" > gpurun_out/cfg_r2g.log
for cfg in "FM_FUSE=0" "FM_FUSE=1" "FM_FUSE=0" "FM_FUSE=1"; do
  echo "== $cfg" >> gpurun_out/ab_r2g.log
  env $cfg timeout 300 python bench.py --no-cpu-baseline --no-erode --steps 10 --warmup 3 2>&1 | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print(d['value'], d['e2e']['value'], d['parity']['ok'], r['share_of_step'], r['ms_per_launch'], d['max_abs_deviation'])" >> gpurun_out/ab_r2g.log 2>&1
done
for cfg in "FM_FUSE=0" "FM_FUSE=1"; do
  n=$(echo $cfg | tr ' =' '__')
  env $cfg timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k regex:"tile128|tonal_kernel" -s 2 -c 20 --csv \
    python bench.py --images 8 --steps 1 --warmup 1 --no-cpu-baseline --no-erode --no-verify > gpurun_out/ncu_r2g_$n.csv 2>&1
done
for c in c1 c2; do
timeout 600 ncu --set full --clock-control none -s 20 -c 4 -o /tmp/prof_r2g_$c \
   python scripts/bench_configs.py --only $c --modes dilate --reps 3 > gpurun_out/ncu_r2g_$c.log 2>&1
ncu -i /tmp/prof_r2g_$c.ncu-rep --page raw --csv > gpurun_out/ncu_r2g_${c}_raw.csv 2>&1
done
