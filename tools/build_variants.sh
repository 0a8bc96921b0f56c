#!/bin/bash
# Build tuning/experiment variants of the library into build/variants/ (not used by the product).
# usage: tools/build_variants.sh name:"-DFLAG=1 -DOTHER" ...
cd "$(dirname "$0")/.."
rm -rf build/variants; mkdir -p build/variants
build() { name=$1; shift; nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -shared -Xcompiler -fPIC -Xptxas -v -Iinclude "$@" -o build/variants/$name.so paper_1705_09907_b200/csrc/hdg_capi.cu 2>build/variants/$name.log & }
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}; [ "$name" = "$spec" ] && flags=""
  build $name $flags
done
wait
ls build/variants/*.so
