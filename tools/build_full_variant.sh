#!/bin/bash
# Builds a complete alternative library (all translation units) with extra
# defines, for layout-changing experiments (e.g. PBDR_KP). Usage: NAME "DEFINES"
set -e
cd "$(dirname "$0")/.."
name=$1; defs=$2
out=build/variants/full_$name; mkdir -p $out
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -lineinfo --fmad=false -Xcompiler -fPIC -Iinclude -Ipaper_2603_14634_b200/csrc $defs"
for f in pbdr_kernels pbdr_sort pbdr_engine pbdr_mesh; do $NV -c paper_2603_14634_b200/csrc/$f.cu -o $out/$f.o -Xptxas -v 2>&1 | grep -A2 "k_iteration" | grep -E "Used|spill" || true; done
for f in pbdr_scene pbdr_errors pbdr_dropin; do g++ -std=c++17 -O3 -fPIC -ffp-contract=off -Iinclude -Ipaper_2603_14634_b200/csrc -I/usr/local/cuda/include $defs -c paper_2603_14634_b200/csrc/$f.cpp -o $out/$f.o; done
$NV -shared -o build/variants/lib_$name.so $out/*.o -lcudart
