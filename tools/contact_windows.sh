#!/bin/bash
# Contact-rich windows of the pile configs (bench.py --preroll): the default
# bench window (frames 4-8) is free flight; these time three frames after the
# piles have landed.
for spec in "3 300" "4 150" "5 100"; do set -- $spec
  timeout 900 python bench.py --config $1 --preroll $2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e | python -c "
import json,sys
d=json.loads(sys.stdin.readline())
r=d['roofline']
print('C$1 frames', d['config']['timed_frames'], 'value=%.3e' % d['value'], 'frame_ms=%.2f' % d['ms_per_step'],
      'substep_frac=%.3f' % r['whole_substep_frac'], {k: round(v, 2) for k, v in r['per_kernel_ms_per_frame'].items()})"
done
