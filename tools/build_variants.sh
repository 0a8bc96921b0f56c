#!/bin/bash
# Build tuning/experiment variants of the library into build/variants/ (not used by the product).
cd "$(dirname "$0")/.."
rm -rf build/variants; mkdir -p build/variants
build() { name=$1; shift; nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -shared -Xcompiler -fPIC -Xptxas -v -Iinclude "$@" -o build/variants/$name.so paper_1705_09907_b200/csrc/hdg_capi.cu 2>build/variants/$name.log & }
build base
build f3_5 -DHDG_F3_MAXN1=5
build f3_5_m1 -DHDG_F3_MAXN1=5 -DHDG_MINB=1
build f3_3 -DHDG_F3_MAXN1=3
wait
ls build/variants/*.so
