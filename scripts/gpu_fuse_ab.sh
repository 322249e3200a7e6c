#!/bin/bash
# A/B of the fused tonal step: bench lines with FM_FUSE=0/1 and chunkings, plus GPU parity tests
TAG=${1:-fuse}
mkdir -p gpurun_out
python -c "from paper_2305_03018_b200 import build; build.build()" > gpurun_out/build_$TAG.log 2>&1
timeout 900 python -m pytest tests/test_gpu_bench_parity.py tests/test_gpu_parity.py tests/test_gpu_fuzz.py -x -q -p no:cacheprovider > gpurun_out/tests_$TAG.log 2>&1
echo "rc=$?" >> gpurun_out/tests_$TAG.log
for cfg in "FM_FUSE=0" "FM_FUSE=1" "FM_FUSE=1 FM_FUSE_KCH=7" "FM_FUSE=1 FM_FUSE_KCH=10" "FM_FUSE=1 FM_DISCARD=0" "FM_FUSE=0" "FM_FUSE=1"; do
  echo "== $cfg" >> gpurun_out/ab_$TAG.log
  env $cfg timeout 300 python bench.py --no-cpu-baseline --no-erode --steps 10 --warmup 3 2>&1 | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print(d['value'], d['e2e']['value'], d['parity']['ok'], r['share_of_step'], r['ms_per_launch'], d['max_abs_deviation'])" >> gpurun_out/ab_$TAG.log 2>&1
done
