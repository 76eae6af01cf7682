run() { timeout 300 env "$@" 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['env'], d['apply_us'])"; }
for mb in 5 6 7; do for r in 1 2 4; do
run MO_B200_JTJ=lc MO_B200_BM=bm8 MO_B200_JTJ9_MINB=$mb MO_B200_JTJ8_R=$r python scripts/exp/ktime.py arap_warp 8192
done; done
run MO_B200_JTJ=lc MO_B200_BM=bm8 MO_B200_JTJ8_NBUF=8 python scripts/exp/ktime.py arap_warp 8192
