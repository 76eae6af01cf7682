timeout 1200 python -m pytest tests -m gpu -q --timeout 600 2>&1 | tail -1
for c in "--config poisson" "--config poisson" "" "" "--config sfs" "--config sfs" "--size 8192" "--config poisson --size 8192" "--config arap_mesh"; do python bench.py $c --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], round(d['value'],4), d['roofline']['kernel'][16:34], round(d['roofline']['avg_launch_us'],2), 'jtf', round(d['roofline_jtf']['avg_launch_us'],2))"; done
