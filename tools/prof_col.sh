#!/bin/bash
# ncu --set full of one explicit_col launch (stage given by --launch-skip) + SASS page
# usage: tools/prof_col.sh <tag> <skip>   (k_ecol launches per step: stage0, stage1, stage2)
tag=$1; skip=${2:-4}
ncu --set full --import-source on --clock-control none -k regex:^k_ecol2?$ --launch-skip $skip --launch-count 1 -f \
    -o gpurun_out/${tag} python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${tag}_ncu.log 2>&1
ncu -i gpurun_out/${tag}.ncu-rep --page raw --csv > gpurun_out/${tag}_raw.csv
ncu -i gpurun_out/${tag}.ncu-rep --page source --csv --print-source=sass > gpurun_out/${tag}_src.csv 2>/dev/null
