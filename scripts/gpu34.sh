for vp in 4 2 8 16 0; do export MO_B200_VEC_PER_SM=$vp; for c in "" "--size 8192"; do timeout 600 python bench.py $c --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('vper=$vp', d['config']['workload'], round(d['value'],4), round(d['roofline']['avg_launch_us'],2), round(d['roofline']['pcg_update_avg_us'],2))"; done; done
