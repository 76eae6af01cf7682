for c in "poisson 8192" "poisson 512"; do timeout 300 python scripts/exp/ktime.py $c 2>&1 | grep '^{'; done
timeout 300 env MO_B200_NO_TILE_LIST=1 python scripts/exp/ktime.py poisson 8192 2>&1 | grep '^{'
timeout 600 python bench.py --config poisson --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['avg_launch_us'], d['roofline_jtf']['avg_launch_us'])"
timeout 900 python -m pytest tests/test_golden_gpu.py tests/test_fullsize_gpu.py tests/test_shard_gpu.py -m gpu -q -p no:cacheprovider -x 2>&1 | tail -2
