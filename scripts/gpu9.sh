timeout 900 python -m pytest tests/test_shard_gpu.py -q --timeout 300 -x 2>&1 | tail -30
timeout 900 python -m pytest tests -m gpu -q --timeout 300 2>&1 | tail -4
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench9.json 2> gpurun_out/bench9.err; tail -3 gpurun_out/bench9.err; python -c "
import json; d=json.load(open('gpurun_out/bench9.json')); print(d['value'], d['roofline']['avg_launch_us'], d['roofline']['pcg_update_avg_us'], d['e2e']['value'], d['gpu_launches'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 300 -c 200 --csv --log-file gpurun_out/launches9_mesh.csv python bench.py --config arap_mesh --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
