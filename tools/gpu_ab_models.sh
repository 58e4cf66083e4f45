# per-unit times of zoo models, A (build/ab) vs B (in-tree)
for m in "$@"; do
  for lib in A B; do
    if [ $lib = A ]; then export WLFUSE_LIB_AB=build/ab/libwlfuse.so; else unset WLFUSE_LIB_AB; fi
    timeout 300 python bench.py --model $m --skip-cpu --steps 10 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); u=d['units']
print('$lib', '$m', round(d['value']), {k:v for k,v in u.items() if k in ('s2b0','s3b0')})"
  done
done
