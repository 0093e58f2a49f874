#!/bin/bash
# The pile configs over their own step counts (BASELINE.json: C3 500 frames,
# C4 200, C5 100): every frame after 3 warm-up frames is timed on the device;
# `tail` is the last 20 frames (contact-rich), `whole` frames 3..end, `head`
# the frames before the tail window. Clocks are sampled over the tail window.
for c in ${@:-3 4 5}; do
  timeout 1500 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-secondary | python -c "
import json,sys
d=json.loads(sys.stdin.readline())
r=d['roofline']
print('C$c', 'N=%d' % d['config']['particles_per_gpu'], 'tail', d['config']['timed_frames'].split(' ')[0], 'value=%.3e' % d['value'],
      'ms/frame=%.2f' % d['ms_per_step'], 'substep_frac=%.3f' % r['whole_substep_frac'],
      'whole %s value=%.3e' % (d['runs']['whole_run']['frames'], d['runs']['whole_run']['value']),
      'head %s value=%.3e' % (d['runs']['before_window']['frames'], d['runs']['before_window']['value']),
      'iter_frac=%.3f' % r['frac'], {k: round(v, 2) for k, v in r['per_kernel_ms_per_frame'].items()}, 'clocks', d['clocks'])"
done
