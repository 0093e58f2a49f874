#!/bin/bash
# Whole runs of the pile configs: frames 4 to the config's own step count
# (BASELINE.json: C3 500 steps, C4 200, C5 100), after 3 warm-up frames.
for spec in "3 497" "4 197" "5 97"; do set -- $spec
  timeout 1500 python bench.py --config $1 --steps $2 --warmup 3 --no-cpu-baseline --no-e2e | python -c "
import json,sys
d=json.loads(sys.stdin.readline())
print('C$1 whole run frames', d['config']['timed_frames'], 'value=%.3e' % d['value'], 'ms/frame=%.2f' % d['ms_per_step'],
      'substep_frac=%.3f' % d['roofline']['whole_substep_frac'])"
done
