#!/bin/bash
# usage: bash scripts/gpu_round.sh TAG [what...]
#   what: peak | tests | benchparity | bench | bench_u8 | profile | configs  (default: tests bench)
TAG=${1:-run}; shift
WHAT=${@:-tests bench}
mkdir -p gpurun_out
python -c "from paper_2305_03018_b200 import build; build.build()" > gpurun_out/build_$TAG.log 2>&1
for w in $WHAT; do
  case $w in
    peak)
      nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp32_peak scripts/micro/fp32_peak.cu && \
        timeout 120 /tmp/fp32_peak > gpurun_out/fp32_peak_$TAG.json 2>&1 ;;
    tests)
      timeout 1500 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/tests_$TAG.log 2>&1
      echo "tests_rc=$?" >> gpurun_out/tests_$TAG.log ;;
    benchparity)
      timeout 900 python -m pytest tests/test_gpu_bench_parity.py -x -q -p no:cacheprovider > gpurun_out/benchparity_$TAG.log 2>&1
      echo "rc=$?" >> gpurun_out/benchparity_$TAG.log ;;
    bench)
      timeout 1200 python bench.py > gpurun_out/bench_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/bench_$TAG.log ;;
    bench_u8)
      timeout 900 python bench.py --out-dtype u8 --no-cpu-baseline > gpurun_out/bench_u8_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/bench_u8_$TAG.log ;;
    ref)
      timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/ref_$TAG.log ;;
    profile)
      bash scripts/gpu_profile.sh $TAG ;;
    configs)
      timeout 900 python scripts/bench_configs.py > gpurun_out/configs_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/configs_$TAG.log ;;
  esac
done
