run() { timeout 300 env "$@" 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['env'], d['apply_us'], d['normal_us'])"; }
run MO_B200_JTJ=lc MO_B200_BM=bm8 python scripts/exp/ktime.py arap_warp 8192
run MO_B200_JTJ=lc MO_B200_BM=bm8 MO_B200_JTJ9_TMA=1 python scripts/exp/ktime.py arap_warp 8192
run MO_B200_JTJ=lc MO_B200_BM=bm8 MO_B200_JTJ9_TMA=1 MO_B200_JTJ8_NBUF=8 python scripts/exp/ktime.py arap_warp 8192
run MO_B200_JTJ=lc MO_B200_BM=bm8 MO_B200_JTJ9_TMA=1 MO_B200_JTJ9_MINB=0 python scripts/exp/ktime.py arap_warp 8192
run MO_B200_JTJ=lc MO_B200_BM=bm8 MO_B200_JTJ9_TMA=1 MO_B200_JTJ8_R=2 python scripts/exp/ktime.py arap_warp 8192
run MO_B200_JTJ=lc MO_B200_BM=bm8 MO_B200_JTJ9_TMA=1 python scripts/exp/ktime.py arap_warp 1024
MO_B200_JTJ=lc MO_B200_JTJ9_TMA=1 timeout 900 python -m pytest tests/test_golden_gpu.py -m gpu -q -p no:cacheprovider -k "variant_parity and lc" 2>&1 | tail -2
