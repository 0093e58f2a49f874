#!/bin/bash
# A/B of library builds on saved contact-rich states (round-2 series): saves
# the states once with the in-tree library, then times every build on the
# identical state and prints ms/frame, the iteration and neighbour-search
# share and a hash of the result (builds that only reorganise work must agree).
#   bash tools/build_variants.sh cb2 "-DPBDR_COOP_BATCH=2" col2 "-DPBDR_CAND_COLUMNS=2"
#   bash tools/ab_states.sh 5:45,5:60,5:80,3:480 build/variants/lib_col2.so build/variants/lib_cb2.so
states=$1; shift
mkdir -p gpurun_out
python tools/ab_landed.py --prep --states $states
for rep in 1 2; do
  for lib in paper_2603_14634_b200/lib/libpbdr_gpu.so "$@"; do
    PBDR_LIB_PATH=$PWD/$lib python tools/ab_landed.py --states $states
  done
done
