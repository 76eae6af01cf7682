python - <<'PY'
import torch
p=torch.cuda.get_device_properties(0); print(p.name, 'L2', p.L2_cache_size)
import ctypes
rt=ctypes.CDLL('libcudart.so') if False else None
PY
nvidia-smi -q | grep -i -A2 "l2\|persist" | head -10
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 2>&1 | tail -2
for c in "" "--config poisson" "--config sfs" "--config arap_mesh"; do for v in 0 1; do if [ $v = 1 ]; then export MO_B200_NO_L2PERSIST=1; else unset MO_B200_NO_L2PERSIST; fi; timeout 600 python bench.py $c --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('nopersist=$v', d['config']['workload'], round(d['value'],4), round(d['roofline']['avg_launch_us'],2), round(d['roofline']['frac'],3), round(d['roofline']['pcg_update_avg_us'],2), round(d['e2e']['value'],3), d['gpu_launches'])"; done; done
