run() {
  cp ab_libs/$1.so paper_1712_04048_b200/libcavs.so
  timeout 200 python bench.py --no-cpu-baseline --no-e2e --steps 20 --warmup 3 2>&1 | tail -1 > gpurun_out/b_$1.json
  python -c "
import json; b=json.load(open('gpurun_out/b_$1.json')); print('$1 $2', round(b['value']), round(b['ms_per_step'],4), {k: round(v['ms_per_step'],4) for k,v in b['phases'].items()})"
}
for v in ${VARIANTS}; do run $v; done
