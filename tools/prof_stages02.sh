#!/bin/bash
# E stage 0 and 2 launches (k_explicit2 launch 4 and 6 of bench --steps 1 --warmup 3), raw pages only
python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/p02_plain.log 2>&1 || exit 1
for sk in 3 5; do
  ncu --set full --clock-control none -k regex:k_explicit2 --launch-skip $sk --launch-count 1 -f -o gpurun_out/p02_$sk \
      python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/p02_ncu_$sk.log 2>&1
  ncu -i gpurun_out/p02_$sk.ncu-rep --page raw --csv > gpurun_out/p02_${sk}_raw.csv 2>/dev/null
  rm -f gpurun_out/p02_$sk.ncu-rep
done
ls gpurun_out
