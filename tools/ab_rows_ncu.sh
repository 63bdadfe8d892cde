# per-launch durations of k_rows (FC fwd, cfg5) for A/B library variants (ncu, warm caches)
for v in ${VARIANTS:-rows_pair rows_noepi rows_notma rows_nomma}; do
  cp ab_libs/$v.so paper_1712_04048_b200/libcavs.so
  for P in 1 0; do
    CAVS_ROWS_PAIR=$P timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_active.avg \
      --cache-control none --clock-control none -k regex:k_rows -c 8 --csv --log-file gpurun_out/abr.csv \
      python bench.py --config cfg5 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --pool 1 --no-flush > /dev/null 2>&1
    python -c "
import csv,sys
rows=[r for r in csv.reader(open('gpurun_out/abr.csv')) if len(r)>5 and not r[0].startswith('==')]
hdr=rows[0]; iid=hdr.index('ID'); ik=hdr.index('Kernel Name'); im=hdr.index('Metric Name'); iv=hdr.index('Metric Value'); ig=hdr.index('Grid Size')
d={}
for r in rows[1:]:
  d.setdefault(r[iid],{})[r[im]]=r[iv]; d[r[iid]]['k']=r[ik][:16]; d[r[iid]]['g']=r[ig]
print('$v pair=$P', ' | '.join(f\"{v['k'][9:16]} g{v['g']} {float(v['gpu__time_duration.sum'])/1e3:.1f}us tp{float(v['sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active']):.0f}%\" for v in list(d.values())[:4]))
"
  done
done
