python tools/near_fraction.py
for c in 3 4 5; do
  for bp in 1 0; do
    PBDR_BROADPHASE=$bp timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e | python -c "
import json,sys
d=json.loads(sys.stdin.readline()); r=d['roofline']; k=r['per_kernel_ms_per_frame']
print('C$c bp=$bp value=%.3e frame=%.2f' % (d['value'], d['ms_per_step']), {x: round(v,2) for x,v in k.items()})"
  done
done
