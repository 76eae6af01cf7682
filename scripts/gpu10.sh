timeout 900 python -m pytest tests -m gpu -q --timeout 300 2>&1 | tail -4
timeout 300 python bench.py --config arap_mesh --steps 3 --warmup 2 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], d['value'], d['roofline']['avg_launch_us'], d['roofline']['pcg_update_avg_us'], d['e2e']['value'])"
timeout 600 python bench.py --size 8192 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench10_8192.json 2> gpurun_out/bench10_8192.err; tail -2 gpurun_out/bench10_8192.err; python -c "
import json; d=json.load(open('gpurun_out/bench10_8192.json')); print(d['config']['workload'], d['value'], d['roofline'], d['e2e']['value'])"
timeout 600 python bench.py --config poisson --size 8192 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench10_p8192.json 2> gpurun_out/bench10_p8192.err; tail -2 gpurun_out/bench10_p8192.err; python -c "
import json; d=json.load(open('gpurun_out/bench10_p8192.json')); print(d['config']['workload'], d['value'], d['roofline'], d['e2e']['value'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 300 -c 200 --csv --log-file gpurun_out/launches10_mesh.csv python bench.py --config arap_mesh --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mo_gather_jtj -s 25 -c 1 -o gpurun_out/prof_jtj10_8192 python bench.py --size 8192 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu10.log 2>&1; tail -1 gpurun_out/ncu10.log
