timeout 1200 python -m pytest tests -m gpu -q --timeout 600 2>&1 | tail -2
for v in 0 1; do if [ $v = 1 ]; then export MO_B200_NO_CONSUMER=1; else unset MO_B200_NO_CONSUMER; fi; for c in "" "--config sfs" "--config poisson" "--size 8192"; do python bench.py $c --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('nocons=$v', d['config']['workload'], round(d['value'],4), round(d['roofline']['avg_launch_us'],2), round(d['roofline']['pcg_update_avg_us'],2), d['config']['final_cost'])"; done; done
