timeout 900 python -m pytest tests -m gpu -q --timeout 200 2>&1 | tail -4
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench8.json 2> gpurun_out/bench8.err; tail -3 gpurun_out/bench8.err; python -c "
import json; d=json.load(open('gpurun_out/bench8.json')); print(d['value'], d['roofline']['avg_launch_us'], d['roofline']['pcg_update_avg_us'], d['e2e']['value'], d['gpu_launches'])"
for c in poisson sfs arap_mesh; do timeout 300 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], d['value'], d['roofline']['avg_launch_us'], d['roofline']['pcg_update_avg_us'], d['e2e']['value'])"; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 200 -c 300 --csv --log-file gpurun_out/launches8.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mo_gather_jtj -s 40 -c 1 -o gpurun_out/prof_jtj8 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu8.log 2>&1; tail -1 gpurun_out/ncu8.log
