#!/bin/bash
# build a variant of liblrbms.so with extra -D flags: tools/build_variant.sh NAME "-DFOO=1 -DBAR=2"
set -e
cd "$(dirname "$0")/.."
mkdir -p variants
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared $2 \
  -o variants/$1.so paper_1405_2810_b200/csrc/lrbms.cu
