#!/bin/bash
# Builds alternative libpbdr_gpu.so builds (pbdr_kernels.cu with extra -D
# defines) into build/variants/ for A/B timing (tools/ab_landed.py with
# PBDR_LIB_PATH). They link the package's libpbdr_host.so.
# Usage: tools/build_variants.sh NAME "EXTRA NVCC DEFINES" [NAME DEFINES ...]
set -e
cd "$(dirname "$0")/.."
mkdir -p build/variants
while [ $# -ge 2 ]; do
  name=$1; defs=$2; shift 2
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -lineinfo --fmad=false \
    -Xcompiler -fPIC,-ffp-contract=off $defs -Xptxas -v -Iinclude -Ipaper_2603_14634_b200/csrc \
    -c paper_2603_14634_b200/csrc/pbdr_kernels.cu -o build/variants/k_$name.o 2> build/variants/k_$name.ptxas.txt
  grep -A2 "k_iterationILi4ELb0ELb0" build/variants/k_$name.ptxas.txt | grep -E "Used|spill" | sed "s/^/$name: /" || true
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/variants/lib_$name.so \
    build/variants/k_$name.o build/obj/pbdr_sort.o build/obj/pbdr_engine.o build/obj/pbdr_mesh.o build/obj/pbdr_slab.o build/obj/pbdr_dropin.o \
    -Lpaper_2603_14634_b200/lib -lpbdr_host -lcudart -lnccl -Xlinker -rpath,'$ORIGIN/../../paper_2603_14634_b200/lib'
done
