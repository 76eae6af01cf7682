for c in "" "--config sfs" "--config poisson" "--size 8192" "--config arap_mesh"; do python bench.py $c --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], round(d['value'],4), round(d['roofline']['avg_launch_us'],2), round(d['roofline']['pcg_update_avg_us'],2), d['config']['final_cost'])"; done
