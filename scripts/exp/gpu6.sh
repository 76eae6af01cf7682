timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo tests_rc=$?
tail -8 gpurun_out/gputest.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo bench_rc=$?; tail -c 1500 gpurun_out/bench.log
