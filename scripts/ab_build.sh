#!/bin/bash
# usage: bash scripts/ab_build.sh NAME — build the working tree and keep the library as _build/ab_NAME.so (FM_LIB A/B runs)
set -e
cd "$(dirname "$0")/.."
python -m paper_2305_03018_b200.build > /dev/null
cp paper_2305_03018_b200/_build/libfftmorph_b200.so paper_2305_03018_b200/_build/ab_$1.so
echo paper_2305_03018_b200/_build/ab_$1.so
