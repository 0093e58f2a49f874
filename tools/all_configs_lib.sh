#!/bin/bash
# all_configs.sh against an alternative library: tools/all_configs_lib.sh LIB [configs...]
lib=$1; shift
cfgs=${@:-1 2 3 4 5}
for c in $cfgs; do
  PBDR_LIB_PATH=$PWD/$lib timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e | python -c "
import json,sys
d=json.loads(sys.stdin.readline())
r=d['roofline']
print('C$c', 'value=%.3e' % d['value'], 'frame_ms=%.2f' % d['ms_per_step'], 'iter_frac=%.3f' % r['frac'], 'substep_frac=%.3f' % r['whole_substep_frac'], 'iter_ms=%.2f' % r['per_kernel_ms_per_frame']['iteration'])"
done
