timeout 900 python -m pytest tests -m gpu -q --timeout 200 -x 2>&1 | tail -15
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench3.json 2> gpurun_out/bench3.err; tail -3 gpurun_out/bench3.err; cat gpurun_out/bench3.json
for c in poisson sfs arap_mesh; do timeout 300 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline 2>&1 | tail -1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 200 -c 300 --csv --log-file gpurun_out/launches3.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; wc -l gpurun_out/launches3.csv
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mo_gather_jtj -s 40 -c 1 -o gpurun_out/prof_jtj3 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu3.log 2>&1; tail -2 gpurun_out/ncu3.log
timeout 600 ncu --set full --clock-control none -k regex:k_pcg_update -s 40 -c 1 -o gpurun_out/prof_upd3 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu3u.log 2>&1; tail -2 gpurun_out/ncu3u.log
