for cfg in 4 5 3; do
for lib in paper_2603_14634_b200/lib/libpbdr_gpu.so build/variants/lib_w4.so paper_2603_14634_b200/lib/libpbdr_gpu.so build/variants/lib_w4.so; do
  PBDR_LIB_PATH=$PWD/$lib timeout 300 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('cfg $cfg $lib value %.4e iter_ms %.4f' % (d['value'], d['roofline']['avg_launch_ms']))"
done; done
