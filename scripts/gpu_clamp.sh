#!/bin/bash
# usage: bash scripts/gpu_clamp.sh TAG — gpu tests, per-config table with and without the clamp bound
TAG=${1:-run}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu_$TAG.log
timeout 600 python scripts/bench_configs.py > gpurun_out/configs_$TAG.log 2>&1; echo rc=$? >> gpurun_out/configs_$TAG.log
FM_RANGE_TAPS=0 timeout 600 python scripts/bench_configs.py > gpurun_out/configs_noclamp_$TAG.log 2>&1; echo rc=$? >> gpurun_out/configs_noclamp_$TAG.log
