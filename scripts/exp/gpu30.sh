b() { timeout 600 env "$@" python bench.py $ARGS --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$ARGS', '$*', d['value'], r['avg_launch_us'], d['roofline_jtf']['avg_launch_us'], r.get('pcg_update_avg_us'))"; }
ARGS="--config poisson" b MO_B200_X=1
ARGS="--config poisson --size 8192" b MO_B200_X=1
ARGS="--config sfs" b MO_B200_X=1
timeout 1500 python -m pytest tests/test_golden_gpu.py tests/test_api_gpu.py tests/test_fullsize_gpu.py tests/test_pcg_gpu.py -m gpu -q -p no:cacheprovider -x -k "poisson or rebound or golden_case or sfs or pcg" 2>&1 | tail -2
