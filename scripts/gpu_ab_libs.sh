#!/bin/bash
# usage: bash scripts/gpu_ab_libs.sh TAG ROUNDS name1 name2 ... — interleaved c5 bench of _build/ab_<name>.so libraries
TAG=$1; R=$2; shift 2
args=()
for r in $(seq $R); do for n in "$@"; do args+=("FM_LIB=paper_2305_03018_b200/_build/ab_$n.so"); done; done
bash scripts/gpu_benchab.sh $TAG "${args[@]}"
