#!/bin/bash
# A/B of whole libraries on the bench configs: tools/ab_libs.sh "CONFIGS" LIB...
# (each library twice, interleaved, 3 timed frames after 3 warm-up frames).
cfgs=$1; shift
for cfg in $cfgs; do
  for rep in 1 2; do
    for lib in "$@"; do
      PBDR_LIB_PATH=$PWD/$lib timeout 300 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null |
        python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('cfg $cfg $lib value %.4e iter_ms %.4f' % (d['value'], d['roofline']['avg_launch_ms']))"
    done
  done
done
