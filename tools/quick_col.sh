#!/bin/bash
# dev-library A/B + bench (N=4 experiment build): tools/quick_col.sh <tag>
export HEVI_LIB=paper_1702_04316_b200/_lib/libhevi_dev.so
timeout 120 python tools/col_ab.py 9 7 3 2>&1 | tail -2
python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/$1.json 2> gpurun_out/$1.err
tail -2 gpurun_out/$1.err
python -c "
import json; d=json.loads(open('gpurun_out/$1.json').read().strip().split(chr(10))[-1]); print(d['ms_per_step']); print(json.dumps({k: v['ms'] for k, v in d['kernels'].items()}))"
