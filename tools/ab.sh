#!/bin/bash
# usage: tools/ab.sh tag1 tag2 ...   A/B of experiment builds (tools/dev_build.sh):
# quick bench + the N=4 3D parity cases per library, twice in alternating order
for rep in 1 2; do
for tag in "$@"; do
    lib=$PWD/paper_1702_04316_b200/_lib/libhevi_$tag.so
    echo "== $tag"
    HEVI_LIB=$lib bash tools/quick_bench.sh
    if [ $rep = 1 ]; then
        HEVI_LIB=$lib python -m pytest tests/test_gpu_parity.py -q -k "box3d_n4 and (steps or rhs)" 2>&1 | tail -1
    fi
done
done
