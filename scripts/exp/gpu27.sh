b() { timeout 600 env "$@" python bench.py $ARGS --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$ARGS', '$*', d['value'], r['avg_launch_us'], r['frac'], r.get('pcg_update_avg_us'))"; }
ARGS="" b MO_B200_X=1
ARGS="--config poisson --size 8192" b MO_B200_X=1
ARGS="" b MO_B200_NO_GROUP_LIST=1 MO_B200_NO_TILE_LIST=1
