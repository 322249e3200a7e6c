mkdir -p gpurun_out
python -c "from paper_2305_03018_b200 import build; build.build()" > gpurun_out/build_r2r.log 2>&1
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/tests_all_r2r.log 2>&1
echo "rc=$?" >> gpurun_out/tests_all_r2r.log
for v in 1 0 1 0; do echo "== FM_OVERLAP=$v" >> gpurun_out/ab_r2r.log
  FM_OVERLAP=$v timeout 300 python bench.py --no-cpu-baseline --no-erode --steps 10 --warmup 3 2>&1 | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print(d['value'], d['e2e']['value'], d['parity']['ok'], r['share_of_step'], r['ms_per_launch'], d['max_abs_deviation'])" >> gpurun_out/ab_r2r.log 2>&1
done
