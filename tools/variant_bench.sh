#!/bin/bash
# Times the iteration kernel and phase split for the default build and any
# alternative builds given as arguments (paths to .so files).
for lib in paper_2603_14634_b200/lib/libpbdr_gpu.so "$@"; do
  echo "== $lib"
  PBDR_LIB_PATH=$PWD/$lib python tools/phase_timing.py | head -9
  PBDR_LIB_PATH=$PWD/$lib timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('value', d['value'], 'iter_ms', d['roofline']['avg_launch_ms'], 'frac', d['roofline']['frac'], d['roofline']['per_kernel_ms_per_frame'])"
done
