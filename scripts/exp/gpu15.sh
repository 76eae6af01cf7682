run() { timeout 300 env "$@" 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['env'], d['apply_us'])"; }
for mb in 0 4 5; do for nb in 4 8; do
run MO_B200_JTJ=lct MO_B200_BM=bm8 MO_B200_JTJ9_MINB=$mb MO_B200_JTJ8_NBUF=$nb python scripts/exp/ktime.py arap_warp 8192
done; done
run MO_B200_JTJ=lct MO_B200_BM=bm8 MO_B200_JTJ8_NW=2 python scripts/exp/ktime.py arap_warp 8192
