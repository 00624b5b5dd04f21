#!/bin/bash
# BASELINE config 2: explicit RK35 at C=1 vs HEVI ARK2 at C=15 and C=150 (same grid family)
for spec in "cfg5 rk35 1" "cfg5 ark2 15" "cfg5w ark2 150" "cfg1 rk35 1" "cfg1 ark2 15"; do
  set -- $spec
  python bench.py --config $1 --integrator $2 --courant $3 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | python -c "
import json,sys
l=[x for x in sys.stdin.read().splitlines() if x.startswith('{')][-1]; d=json.loads(l)
print('$1', '$2', 'C=$3', 'ms/step %.3f' % d['ms_per_step'], 'DOF/s %.3e' % d['value'], 'sim-s per wall-s %.1f' % d['config']['sim_seconds_per_wall_second'])"
done
