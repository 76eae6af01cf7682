run() { timeout 300 env "$@" python scripts/exp/ktime.py arap_warp 8192 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['env'], d['apply'], d['apply_us'], d['normal'], d['normal_us'])"; }
run MO_B200_JTJ=lct MO_B200_BM=bm8
run MO_B200_JTJ=lct MO_B200_BM=bm8 MO_B200_BM8_MINB=4
run MO_B200_JTJ=lct MO_B200_BM=bm8 MO_B200_BM8_MINB=3
run MO_B200_JTJ=lct MO_B200_BM=bm8 MO_B200_JTJ8_R=1
run MO_B200_JTJ=lct MO_B200_BM=bm8 MO_B200_JTJ8_R=1 MO_B200_JTJ8_NBUF=8
run MO_B200_JTJ=lct MO_B200_BM=bm8 MO_B200_JTJ8_R=4 MO_B200_JTJ8_NBUF=2
run
timeout 300 python scripts/exp/ktime.py arap_warp 1024 2>&1 | grep '^{'
timeout 300 python scripts/exp/ktime.py sfs 2>&1 | grep '^{'
timeout 300 python scripts/exp/ktime.py poisson 8192 2>&1 | grep '^{'
