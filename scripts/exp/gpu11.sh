run() { timeout 300 env "$@" 2>&1 | grep '^{' ; }
for pf in 1 2 3; do for mb in 0 6; do
run MO_B200_JTJ=lc MO_B200_BM=bm8 MO_B200_JTJ9_PF=$pf MO_B200_JTJ8_MINB=$mb python scripts/exp/ktime.py arap_warp 8192
done; done
run MO_B200_JTJ=lc MO_B200_BM=bm8 MO_B200_JTJ9_PF=2 python scripts/exp/ktime.py arap_warp 1024
