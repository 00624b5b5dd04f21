# usage: bash /tmp/ab_run.sh libA libB [libA libB ...] : lib_ab bitwise + bench_libs
L=paper_1702_04316_b200/_lib
HEVI_LIB=$L/libhevi_$1.so timeout 300 python tools/lib_ab.py run gpurun_out/ab_a.npz 2>&1 | tail -1
HEVI_LIB=$L/libhevi_$2.so timeout 300 python tools/lib_ab.py run gpurun_out/ab_b.npz 2>&1 | tail -1
python tools/lib_ab.py cmp gpurun_out/ab_a.npz gpurun_out/ab_b.npz 2>&1 | tail -5
rm -f gpurun_out/ab_*.npz
args=""; for t in "$@"; do args="$args $L/libhevi_$t.so"; done
bash tools/bench_libs.sh $args $args
