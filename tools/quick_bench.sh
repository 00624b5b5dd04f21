#!/bin/bash
# usage: tools/quick_bench.sh [extra bench args]  -- prints ms/step and per-kernel ms
python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline "$@" 2>&1 | python -c "
import json,sys
lines=[l for l in sys.stdin.read().strip().splitlines() if l.startswith('{')]
d=json.loads(lines[-1]); print('ms/step', round(d['ms_per_step'],3), 'DOF/s %.3e' % d['value'], 'frac', d['roofline']['frac'], {k:v['ms'] for k,v in d['kernels'].items()})"
