# bitwise A/B of the dev library against the full build, then the dev-library bench
python tools/lib_ab.py run gpurun_out/ab_old.npz 2>&1 | tail -1
HEVI_LIB=paper_1702_04316_b200/_lib/libhevi_dev.so python tools/lib_ab.py run gpurun_out/ab_new.npz 2>&1 | tail -1
python tools/lib_ab.py cmp gpurun_out/ab_old.npz gpurun_out/ab_new.npz
rm -f gpurun_out/ab_*.npz
bash tools/quick_col.sh ${1:-dev}
