for g in 0 1; do for v in 0 1; do if [ $v = 1 ]; then export MO_B200_NO_L2PERSIST=1; else unset MO_B200_NO_L2PERSIST; fi; if [ $g = 1 ]; then export MO_B200_NOGRAPH=1; else unset MO_B200_NOGRAPH; fi; timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('nograph=$g nopersist=$v', d['config']['workload'], round(d['value'],4), round(d['roofline']['avg_launch_us'],2), round(d['roofline']['pcg_update_avg_us'],2))"; done; done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct --cache-control none --clock-control none -s 400 -c 60 --csv --log-file gpurun_out/launches22.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/launches22.csv')))
hi=next(i for i,r in enumerate(rows) if 'Kernel Name' in r); h=rows[hi]
k=h.index('Kernel Name'); m=h.index('Metric Name'); v=h.index('Metric Value'); idx=h.index('ID')
from collections import defaultdict
d=defaultdict(dict)
for r in rows[hi+1:]:
  d[(r[idx], r[k][:30])][r[m]]=r[v]
for key,val in list(d.items())[:30]: print(key, val)
PY
