#!/bin/bash
# Builds alternative k_iteration builds into build/variants/ for A/B timing.
# Usage: tools/build_variants.sh NAME "EXTRA NVCC DEFINES" [NAME DEFINES ...]
set -e
cd "$(dirname "$0")/.."
mkdir -p build/variants
while [ $# -ge 2 ]; do
  name=$1; defs=$2; shift 2
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -lineinfo --fmad=false \
    -Xcompiler -fPIC $defs -Xptxas -v -Iinclude -Ipaper_2603_14634_b200/csrc \
    -c paper_2603_14634_b200/csrc/pbdr_kernels.cu -o build/variants/k_$name.o 2>&1 | grep -A2 k_iteration | grep -E "Used|spill" || true
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/variants/lib_$name.so \
    build/variants/k_$name.o build/obj/pbdr_sort.o build/obj/pbdr_engine.o build/obj/pbdr_mesh.o build/obj/pbdr_scene.o \
    build/obj/pbdr_errors.o build/obj/pbdr_dropin.o -lcudart
done
