nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv; nproc
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -4
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 2>&1 | tail -6
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench12.json 2> gpurun_out/bench12.err; tail -3 gpurun_out/bench12.err; cat gpurun_out/bench12.json
for c in "--config poisson" "--config sfs" "--config arap_mesh" "--size 8192" "--config poisson --size 8192"; do timeout 600 python bench.py $c --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], round(d['value'],4), round(d['roofline']['avg_launch_us'],2), round(d['roofline']['frac'],3), round(d['roofline']['pcg_update_avg_us'],2), round(d['e2e']['value'],3), d['gpu_launches'])"; done
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref12.json 2>&1; tail -1 gpurun_out/bench_ref12.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 300 -c 300 --csv --log-file gpurun_out/launches12.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; python scripts/launches.py gpurun_out/launches12.csv
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mo_gather_jtj -s 25 -c 1 -o gpurun_out/prof_jtj12_8192 python bench.py --size 8192 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu12.log 2>&1; tail -1 gpurun_out/ncu12.log
