#!/bin/bash
# ncu --set full of one k_solve2 launch (first timed step's stage-0 solve) + SASS page
# usage: tools/prof_solve.sh <tag>   (uses HEVI_LIB if set)
tag=$1
ncu --set full --import-source on --clock-control none -k regex:^k_solve2$ --launch-skip 6 --launch-count 1 -f \
    -o gpurun_out/${tag} python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${tag}_ncu.log 2>&1
ncu -i gpurun_out/${tag}.ncu-rep --page raw --csv > gpurun_out/${tag}_raw.csv
ncu -i gpurun_out/${tag}.ncu-rep --page source --csv --print-source=sass > gpurun_out/${tag}_src.csv 2>/dev/null
rm -f gpurun_out/${tag}.ncu-rep
