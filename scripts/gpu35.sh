for ch in 0 6 14 22 30 38 46 62 70 94; do export MO_B200_CHUNK=$ch; [ $ch = 0 ] && unset MO_B200_CHUNK; MO_B200_JTJ=tma timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('chunk=$ch', d['config']['workload'], round(d['value'],4), round(d['roofline']['avg_launch_us'],2))"; done
