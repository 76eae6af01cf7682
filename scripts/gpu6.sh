timeout 900 python -m pytest tests -m gpu -q --timeout 200 2>&1 | tail -4
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench6.json 2> gpurun_out/bench6.err; tail -3 gpurun_out/bench6.err; python -c "
import json; d=json.load(open('gpurun_out/bench6.json')); print(d['value'], d['roofline']['avg_launch_us'], d['roofline']['pcg_update_avg_us'], d['e2e']['value'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 200 -c 300 --csv --log-file gpurun_out/launches6.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mo_gather_jtj -s 40 -c 1 -o gpurun_out/prof_jtj6 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu6.log 2>&1; tail -1 gpurun_out/ncu6.log
