timeout 1200 python -m pytest tests -m gpu -q --timeout 600 2>&1 | tail -2
for c in "" "--size 8192" "--config poisson" "--config poisson --size 8192" "--config sfs" "--config arap_mesh"; do timeout 600 python bench.py $c --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], round(d['value'],4), d['roofline']['kernel'][:36], round(d['roofline']['avg_launch_us'],2), round(d['e2e']['value'],3), d['gpu_launches'], d['config']['final_cost'])"; done
