#!/bin/bash
# Builds alternative k_iteration register budgets into build/variants/ for A/B timing.
set -e
cd "$(dirname "$0")/.."
mkdir -p build/variants
for mb in "$@"; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -lineinfo --fmad=false \
    -Xcompiler -fPIC -DPBDR_ITER_MINBLOCKS=$mb -Xptxas -v -Iinclude -Ipaper_2603_14634_b200/csrc \
    -c paper_2603_14634_b200/csrc/pbdr_kernels.cu -o build/variants/k$mb.o 2>&1 | grep -A2 k_iteration | grep -E "Used|spill"
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/variants/libpbdr_mb$mb.so \
    build/variants/k$mb.o build/obj/pbdr_sort.o build/obj/pbdr_engine.o build/obj/pbdr_scene.o \
    build/obj/pbdr_errors.o build/obj/pbdr_dropin.o -lcudart
done
