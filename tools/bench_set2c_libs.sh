# set2c bench per library: tools/bench_set2c_libs.sh lib1.so [lib2.so ...]
for L in "$@"; do
  HEVI_LIB=$L python bench.py --set set2c --steps 20 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$L', round(d['ms_per_step'],4), json.dumps({k: v['ms'] for k, v in d['kernels'].items()}))"
done
