timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -x 2>&1 | tail -3
for v in 0 1; do if [ $v = 1 ]; then export MO_B200_NO_BM4=1; else unset MO_B200_NO_BM4; fi; for c in "" "--config sfs" "--config poisson" "--size 8192"; do python bench.py $c --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('nobm4=$v', d['config']['workload'], round(d['value'],4), 'jtf', round(d['roofline_jtf']['avg_launch_us'],2), round(d['roofline_jtf']['frac'],3), d['config']['final_cost'])"; done; done
