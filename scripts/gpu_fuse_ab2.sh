#!/bin/bash
# A/B of the fused tonal step + DRAM bytes of the conv kernel (fused / unfused) by ncu
TAG=${1:-fuse2}
mkdir -p gpurun_out
python -c "from paper_2305_03018_b200 import build; build.build()" > gpurun_out/build_$TAG.log 2>&1
for cfg in "FM_FUSE=0" "FM_FUSE=1" "FM_FUSE=1 FM_DISCARD=0" "FM_FUSE=0" "FM_FUSE=1" "FM_FUSE=1 FM_DISCARD=0"; do
  echo "== $cfg" >> gpurun_out/ab_$TAG.log
  env $cfg timeout 300 python bench.py --no-cpu-baseline --no-erode --steps 10 --warmup 3 2>&1 | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print(d['value'], d['e2e']['value'], d['parity']['ok'], r['share_of_step'], r['ms_per_launch'], d['max_abs_deviation'])" >> gpurun_out/ab_$TAG.log 2>&1
done
for cfg in "FM_FUSE=0" "FM_FUSE=1" "FM_FUSE=1 FM_DISCARD=0"; do
  n=$(echo $cfg | tr ' =' '__')
  env $cfg timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum \
    --clock-control none -k regex:"tile128_kernelIhLb0|tonal_kernel_pipe" -s 2 -c 12 --csv \
    python bench.py --images 8 --steps 1 --warmup 1 --no-cpu-baseline --no-erode --no-verify > gpurun_out/ncu_${TAG}_$n.csv 2>&1
done
