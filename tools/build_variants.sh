#!/bin/bash
# Build tuning/experiment variants of the library into build/variants/ (not used by the product).
cd "$(dirname "$0")/.."
rm -rf build/variants; mkdir -p build/variants
build() { name=$1; shift; nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -shared -Xcompiler -fPIC -Iinclude "$@" -o build/variants/$name.so paper_1705_09907_b200/csrc/hdg_capi.cu 2>build/variants/$name.log & }
build base
build ws_nb2 -DHDG_WS=1 -DHDG_NBUF=2
build ws_nb3_f0 -DHDG_WS=1 -DHDG_NBUF=3 -DHDG_F_MAXN1=0
build ws_nb4_f0 -DHDG_WS=1 -DHDG_NBUF=4 -DHDG_F_MAXN1=0 -DHDG_WS_MINB=1
build ws_nb2_m1 -DHDG_WS=1 -DHDG_NBUF=2 -DHDG_WS_MINB=1
build base_stageonly -DHDG_EXP_NOCOMPUTE -DHDG_EXP_NOOUT
wait
ls build/variants/*.so
