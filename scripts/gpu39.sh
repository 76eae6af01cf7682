for sz in 128 256 512 1024 2048; do timeout 600 python bench.py --size $sz --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$sz', round(d['value'],4), d['roofline']['kernel'][:36], 'apply', round(d['roofline']['avg_launch_us'],2), 'upd+p', round(d['roofline']['pcg_update_avg_us'],2))"; done
