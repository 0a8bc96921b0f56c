#!/bin/bash
# Build tuning/experiment variants of the library into build/variants/ (not used by the product).
cd "$(dirname "$0")/.."
rm -rf build/variants; mkdir -p build/variants
build() { name=$1; shift; nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -shared -Xcompiler -fPIC -Iinclude "$@" -o build/variants/$name.so paper_1705_09907_b200/csrc/hdg_capi.cu 2>build/variants/$name.log & }
build base
build dmma -DHDG_DMMA=1
build dmma_nb2 -DHDG_DMMA=1 -DHDG_NBUF=2
build dmma_computeonly -DHDG_DMMA=1 -DHDG_EXP_NOSTAGE -DHDG_EXP_NOOUT
wait
ls build/variants/*.so
