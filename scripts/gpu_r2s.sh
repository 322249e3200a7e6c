mkdir -p gpurun_out
python -c "from paper_2305_03018_b200 import build; build.build()" > gpurun_out/build_r2s.log 2>&1
FM_FUSE=1 timeout 900 python -m pytest tests/test_gpu_bench_parity.py tests/test_gpu_parity.py tests/test_gpu_fuzz.py -q -p no:cacheprovider > gpurun_out/tests_fused_r2s.log 2>&1
echo "rc=$?" >> gpurun_out/tests_fused_r2s.log
for cfg in "FM_FUSE=0" "FM_FUSE=1" "FM_FUSE=1 FM_DISCARD=0" "FM_FUSE=1 FM_FUSE_KCH=14" "FM_FUSE=0" "FM_FUSE=1"; do
  echo "== $cfg" >> gpurun_out/ab_r2s.log
  env $cfg timeout 300 python bench.py --no-cpu-baseline --no-erode --steps 10 --warmup 3 2>&1 | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print(d['value'], d['e2e']['value'], d['parity']['ok'], r['share_of_step'], r['ms_per_launch'], d['max_abs_deviation'])" >> gpurun_out/ab_r2s.log 2>&1
done
for cfg in "FM_FUSE=0" "FM_FUSE=1" "FM_FUSE=1 FM_FUSE_KCH=14"; do
  n=$(echo $cfg | tr ' =' '__')
  env $cfg timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv python bench.py --profile-step --no-cpu-baseline > gpurun_out/ncu_r2s_$n.csv 2>&1
done
