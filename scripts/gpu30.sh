timeout 1200 python -m pytest tests -m gpu -q --timeout 600 2>&1 | tail -3
for v in 0 1; do if [ $v = 1 ]; then export MO_B200_NO_VFUSE=1; else unset MO_B200_NO_VFUSE; fi; timeout 600 python bench.py --config arap_mesh --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('novfuse=$v', d['config']['workload'], round(d['value'],4), round(d['roofline']['avg_launch_us'],2), round(d['roofline']['pcg_update_avg_us'],2), round(d['e2e']['value'],3), d['gpu_launches'], d['config']['final_cost'])"; done
