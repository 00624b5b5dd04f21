#!/bin/bash
# usage: tools/prof_e.sh <tag> [launch-skip] [extra bench args]
# One `ncu --set full` capture of an explicit-stage launch (default: the 5th
# k_explicit2 launch = E stage 1 of the second step) after a clean bench run.
tag=${1:-e}; skip=${2:-4}; shift 2
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline "$@" > gpurun_out/plain_$tag.log 2>&1 || exit 1
ncu --set full --import-source on --clock-control none -k regex:k_explicit --launch-skip $skip \
    --launch-count 1 -f -o gpurun_out/prof_$tag python bench.py --steps 1 --warmup 3 --no-e2e \
    --no-cpu-baseline "$@" > gpurun_out/ncu_$tag.log 2>&1
