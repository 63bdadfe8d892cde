for v in base spin; do
  cp ab_libs/$v.so paper_1712_04048_b200/libcavs.so
  for pb in 0 1; do
    CAVS_PBWD=$pb timeout 300 python bench.py --steps 20 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v PBWD=$pb', round(d['value']), {k: round(v['ms_per_step']*1000,1) for k,v in d['phases'].items()})"
  done
done
