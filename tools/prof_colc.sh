#!/bin/bash
# ncu of one set2c explicit_colc launch: tools/prof_colc.sh <tag> <skip>
tag=$1; skip=${2:-4}
ncu --set full --import-source on --clock-control none -k regex:^k_ecolc$ --launch-skip $skip --launch-count 1 -f \
    -o gpurun_out/${tag} python bench.py --set set2c --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${tag}_ncu.log 2>&1
ncu -i gpurun_out/${tag}.ncu-rep --page raw --csv > gpurun_out/${tag}_raw.csv
ncu -i gpurun_out/${tag}.ncu-rep --page source --csv --print-source=sass > gpurun_out/${tag}_src.csv 2>/dev/null
rm -f gpurun_out/${tag}.ncu-rep
