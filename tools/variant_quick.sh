for lib in "$@"; do
  echo "== $lib"
  PBDR_LIB_PATH=$PWD/$lib python tools/phase_timing.py | grep -E "phase|bodymath|lifetime|resident"
  PBDR_LIB_PATH=$PWD/$lib timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('value %.3e iter_ms %.4f' % (d['value'], d['roofline']['avg_launch_ms']))"
done
