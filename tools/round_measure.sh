#!/bin/bash
# GPU-box measurement pass: gpu tests, bench (both arms), launch list, ncu
# captures of every explicit stage (k_ecol) and the column solve (k_solve2).
# Outputs in gpurun_out/<tag>_*.
tag=${1:-r02}
[ -z "$SKIP_TESTS" ] && python -m pytest tests -m gpu -q > gpurun_out/${tag}_gputests.log 2>&1
tail -3 gpurun_out/${tag}_gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1
python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err || exit 1
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${tag}_bench_ref.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 3 --warmup 3 --no-e2e \
    --no-cpu-baseline > gpurun_out/${tag}_ncu_launch.log 2>&1
# explicit stages 0, 1, 2 of the first timed step (3 warm-up steps x 3 launches skipped)
ncu --set full --import-source on --clock-control none -k regex:^k_ecol$ --launch-skip 9 \
    --launch-count 3 -f -o gpurun_out/${tag}_e python bench.py --steps 1 --warmup 3 --no-e2e \
    --no-cpu-baseline > gpurun_out/${tag}_ncu_e.log 2>&1
# column solves of the first timed step
ncu --set full --import-source on --clock-control none -k regex:^k_solve2$ --launch-skip 6 \
    --launch-count 2 -f -o gpurun_out/${tag}_s python bench.py --steps 1 --warmup 3 --no-e2e \
    --no-cpu-baseline > gpurun_out/${tag}_ncu_s.log 2>&1
# set2c (flux form): bench line and one explicit stage-1 launch
python bench.py --set set2c --steps 20 --no-e2e > gpurun_out/${tag}_bench_set2c.json 2>&1
ncu --set full --import-source on --clock-control none -k regex:^k_ecolc$ --launch-skip 10 \
    --launch-count 1 -f -o gpurun_out/${tag}_c python bench.py --set set2c --steps 1 --warmup 3 \
    --no-e2e --no-cpu-baseline > gpurun_out/${tag}_ncu_c.log 2>&1
for r in e s c; do
  ncu -i gpurun_out/${tag}_$r.ncu-rep --page raw --csv > gpurun_out/${tag}_${r}_raw.csv 2>/dev/null
  ncu -i gpurun_out/${tag}_$r.ncu-rep --page source --csv --print-source=sass > gpurun_out/${tag}_${r}_src.csv 2>/dev/null
done
gzip -f gpurun_out/${tag}_*_src.csv
rm -f gpurun_out/${tag}_[esc].ncu-rep
tail -1 gpurun_out/${tag}_bench.json | cut -c1-400
