#!/bin/bash
# usage: tools/dev_build.sh <tag> [nvcc -D flags...]  -> paper_1702_04316_b200/_lib/libhevi_<tag>.so
# experiment build: N=4 only (HEVI_DEV_N), for A/B runs via HEVI_LIB
tag=$1; shift
cd "$(dirname "$0")/../paper_1702_04316_b200" || exit 1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
    csrc/hevi.cu -DHEVI_DEV_N=4 "$@" -o _lib/libhevi_$tag.so 2>&1 | grep -E "error|warning: R" | head
