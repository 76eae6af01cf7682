run() { timeout 300 env "$@" 2>&1 | grep '^{' ; }
run MO_B200_JTJ=lc MO_B200_BM=bm8 python scripts/exp/ktime.py arap_warp 8192
run MO_B200_JTJ=lc MO_B200_BM=bm8 MO_B200_NO_BM8C=1 python scripts/exp/ktime.py arap_warp 8192
MO_B200_JTJ=lc MO_B200_BM=bm8 timeout 900 python -m pytest tests/test_golden_gpu.py -m gpu -q -p no:cacheprovider -k "golden_case and fma" 2>&1 | tail -3
MO_B200_JTJ=lc MO_B200_BM=bm8 timeout 900 python -m pytest tests/test_fullsize_gpu.py -m gpu -q -p no:cacheprovider -k "arap_warp_1024 or arap_warp]" 2>&1 | tail -3
timeout 600 python bench.py --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['avg_launch_us'], d['roofline']['frac'], d['roofline_jtf']['kernel'], d['roofline_jtf']['avg_launch_us'], d['roofline_jtf']['frac'])"
