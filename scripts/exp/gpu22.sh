b() { timeout 600 env "$@" python bench.py $ARGS --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$ARGS', d['value'], d['roofline']['avg_launch_us'], d['roofline'].get('pcg_update_avg_us'))"; }

for v in 4 2 1 8; do ARGS="--config poisson" b MO_B200_VEC_PER_SM=$v; done
