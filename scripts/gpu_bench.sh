#!/bin/bash
TAG=${1:-run}
mkdir -p gpurun_out
timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bench_$TAG.log 2>&1; echo bench_rc=$? >> gpurun_out/bench_$TAG.log
