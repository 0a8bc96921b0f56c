#!/bin/bash
# Build tuning/experiment variants of the library into build/variants/ (not used by the product).
cd "$(dirname "$0")/.."
rm -rf build/variants; mkdir -p build/variants
build() { name=$1; shift; nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -shared -Xcompiler -fPIC -Iinclude "$@" -o build/variants/$name.so paper_1705_09907_b200/csrc/hdg_capi.cu 2>build/variants/$name.log & }
build m2 -DHDG_MINB=2
build m1 -DHDG_MINB=1
build m2_nb3_f0 -DHDG_MINB=2 -DHDG_NBUF=3 -DHDG_F_MAXN1=0
build m3_nb2_f0 -DHDG_MINB=3 -DHDG_NBUF=2 -DHDG_F_MAXN1=0
build m1_nb3 -DHDG_MINB=1 -DHDG_NBUF=3
build m2_computeonly -DHDG_MINB=2 -DHDG_EXP_NOSTAGE -DHDG_EXP_NOOUT
build m2_stageonly -DHDG_MINB=2 -DHDG_EXP_NOCOMPUTE -DHDG_EXP_NOOUT
build m2_nb3_f0_stageonly -DHDG_MINB=2 -DHDG_NBUF=3 -DHDG_F_MAXN1=0 -DHDG_EXP_NOCOMPUTE -DHDG_EXP_NOOUT
wait
ls build/variants/*.so
