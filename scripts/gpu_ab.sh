#!/bin/bash
# usage: bash scripts/gpu_ab.sh TAG "VAR=value" — gpu tests, then the per-config table as built and with VAR set
TAG=${1:-run}; AB=${2:-FM_RANGE_TAPS=0}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu_$TAG.log
timeout 600 python scripts/bench_configs.py > gpurun_out/configs_$TAG.log 2>&1; echo rc=$? >> gpurun_out/configs_$TAG.log
env $AB timeout 600 python scripts/bench_configs.py > gpurun_out/configs_ab_$TAG.log 2>&1; echo rc=$? >> gpurun_out/configs_ab_$TAG.log
