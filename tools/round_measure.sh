#!/bin/bash
# GPU-box measurement pass: gpu tests, bench (both arms), launch list, ncu capture
# of the dominant kernel.  Outputs in gpurun_out/<tag>_*.
tag=${1:-r01}
python -m pytest tests -m gpu -q > gpurun_out/${tag}_gputests.log 2>&1
tail -3 gpurun_out/${tag}_gputests.log
python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err || exit 1
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${tag}_bench_ref.json 2>&1
python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${tag}_plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 3 --warmup 3 --no-e2e \
    --no-cpu-baseline > gpurun_out/${tag}_ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_explicit2 --launch-skip 4 \
    --launch-count 1 -f -o gpurun_out/${tag}_e1 python bench.py --steps 1 --warmup 3 --no-e2e \
    --no-cpu-baseline > gpurun_out/${tag}_ncu_full.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_solve2 --launch-skip 2 \
    --launch-count 1 -f -o gpurun_out/${tag}_s python bench.py --steps 1 --warmup 3 --no-e2e \
    --no-cpu-baseline > gpurun_out/${tag}_ncu_s.log 2>&1
# text exports on the box (reports are large): raw metrics + per-line source table
for r in e1 s; do
  ncu -i gpurun_out/${tag}_$r.ncu-rep --page raw --csv > gpurun_out/${tag}_${r}_raw.csv 2>/dev/null
  ncu -i gpurun_out/${tag}_$r.ncu-rep --page source --csv --print-source=cuda,sass > gpurun_out/${tag}_${r}_src.csv 2>/dev/null
done
rm -f gpurun_out/${tag}_s.ncu-rep
gzip -f gpurun_out/${tag}_*_src.csv
cat gpurun_out/${tag}_bench.json | tail -1 | cut -c1-600
