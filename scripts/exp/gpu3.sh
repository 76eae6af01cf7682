run() { timeout 300 env "$@" 2>&1 | grep '^{' ; }
for c in "arap_warp 8192" "poisson 8192"; do
  run MO_B200_JTJ=tma MO_B200_BM=bm4 python scripts/exp/ktime.py $c
  run MO_B200_JTJ=gather MO_B200_BM=prog python scripts/exp/ktime.py $c
  run MO_B200_JTJ=ws MO_B200_BM=bm8 python scripts/exp/ktime.py $c
  run MO_B200_JTJ=ws MO_B200_BM=bm8 MO_B200_JTJ8_R=1 python scripts/exp/ktime.py $c
  run MO_B200_JTJ=ws MO_B200_BM=bm8 MO_B200_JTJ8_R=4 python scripts/exp/ktime.py $c
  run MO_B200_JTJ=ws MO_B200_BM=bm8 MO_B200_JTJ8_NBUF=8 MO_B200_JTJ8_R=1 python scripts/exp/ktime.py $c
  run MO_B200_JTJ=ws MO_B200_BM=bm8 MO_B200_JTJ8_MINB=8 MO_B200_BM8_MINB=6 python scripts/exp/ktime.py $c
  run MO_B200_JTJ=ws MO_B200_BM=bm8 MO_B200_JTJ8_NW=2 python scripts/exp/ktime.py $c
done
