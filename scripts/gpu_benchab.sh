#!/bin/bash
# usage: bash scripts/gpu_benchab.sh TAG "ENV=.." ["ENV=.." ...] — c5 bench line per env setting (A/B), "-" = as built
TAG=$1; shift
mkdir -p gpurun_out
out=gpurun_out/benchab_$TAG.log; : > $out
for e in "$@"; do
  if [ "$e" == "-" ]; then e="FM_NONE=1"; fi
  echo "== $e" >> $out
  env $e timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print(round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'conv_ms', round(r['ms_per_launch'],3), 'planes', round(d['config']['mean_planes_per_tile'],3))" >> $out 2>&1
done
