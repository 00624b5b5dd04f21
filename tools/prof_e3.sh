#!/bin/bash
# ncu --set full of the three explicit stages (k_ecol) of the first timed step,
# raw + SASS source pages: tools/prof_e3.sh <tag>   (uses HEVI_LIB if set)
tag=$1
ncu --set full --import-source on --clock-control none -k regex:^k_ecol$ --launch-skip 9 \
    --launch-count 3 -f -o gpurun_out/${tag}_e python bench.py --steps 1 --warmup 3 --no-e2e \
    --no-cpu-baseline > gpurun_out/${tag}_ncu_e.log 2>&1
ncu -i gpurun_out/${tag}_e.ncu-rep --page raw --csv > gpurun_out/${tag}_e_raw.csv 2>/dev/null
ncu -i gpurun_out/${tag}_e.ncu-rep --page source --csv --print-source=sass > gpurun_out/${tag}_e_src.csv 2>/dev/null
gzip -f gpurun_out/${tag}_e_src.csv
rm -f gpurun_out/${tag}_e.ncu-rep
