MO_B200_JTJ=tma4 timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -k "variant or fullsize or golden" 2>&1 | tail -2
for c in "" "--size 8192" "--config sfs" "--config poisson"; do for v in tma tma4; do MO_B200_JTJ=$v timeout 600 python bench.py $c --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['config']['workload'], round(d['value'],4), d['roofline']['kernel'][:36], round(d['roofline']['avg_launch_us'],2), d['config']['final_cost'])"; done; done
