#!/bin/bash
# One bench line per BASELINE.json config (device-resident value + roofline).
for c in 1 2 3 4 5; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --window head --no-secondary --no-cpu-baseline --no-e2e | python -c "
import json,sys
d=json.loads(sys.stdin.readline())
r=d['roofline']
print('C$c', d['config']['workload'], 'N=%d' % d['config']['particles_per_gpu'], 'value=%.3e' % d['value'],
      'frame_ms=%.2f' % d['ms_per_step'], 'iter_frac=%.3f' % r['frac'], 'substep_frac=%.3f' % r['whole_substep_frac'],
      {k: round(v, 2) for k, v in r['per_kernel_ms_per_frame'].items()}, 'clocks', d['clocks'])"
done
