#!/bin/bash
# Build soa_lab variants: tools/soa_lab_build.sh name:"-DFLAGS" ...  -> build/lab/<name>
cd "$(dirname "$0")/.."
mkdir -p build/lab
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}; [ "$name" = "$spec" ] && flags=""
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Ipaper_1705_09907_b200/csrc -Iinclude -DLAB_N1=${LAB_N1:-5} $flags -o build/lab/$name tools/soa_lab.cu &
done
wait
ls build/lab
