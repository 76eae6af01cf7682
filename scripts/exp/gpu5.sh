run() { timeout 300 env "$@" 2>&1 | grep '^{' ; }
for c in "arap_warp 8192" "arap_warp 1024"; do
  run MO_B200_JTJ=lc python scripts/exp/ktime.py $c
done
timeout 300 python scripts/exp/var_times.py arap_warp 8192 2>&1 | grep -v Warn
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/gputest.log 2>&1; echo tests_rc=$?
tail -5 gpurun_out/gputest.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo bench_rc=$?; tail -c 2500 gpurun_out/bench.log
