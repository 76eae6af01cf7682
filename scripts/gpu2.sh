set -x
nproc; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -m pytest tests/test_api_gpu.py -q -x -k grows 2>&1 | tail -40
timeout 600 python -m pytest tests -m gpu -q --timeout 120 2>&1 | tail -8
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench1.json 2> gpurun_out/bench1.err; tail -3 gpurun_out/bench1.err; cat gpurun_out/bench1.json
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref1.json 2>&1; cat gpurun_out/bench_ref1.json | tail -3
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/launches1.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; wc -l gpurun_out/launches1.csv
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mo_gather_jtj -s 40 -c 1 -o gpurun_out/prof_jtj1 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu1.log 2>&1; tail -3 gpurun_out/ncu1.log
