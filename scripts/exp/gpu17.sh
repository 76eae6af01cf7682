# mask prefetch in the jtj8/9 family: times + parity
for v in lct lc ws; do timeout 300 env MO_B200_JTJ=$v MO_B200_BM=bm8 python scripts/exp/ktime.py arap_warp 8192 2>&1 | grep '^{'; done
timeout 300 python scripts/exp/ktime.py arap_warp 8192 2>&1 | grep '^{'
timeout 300 python scripts/exp/ktime.py arap_warp 1024 2>&1 | grep '^{'
timeout 300 python scripts/exp/ktime.py sfs 2>&1 | grep '^{'
timeout 900 python -m pytest tests/test_golden_gpu.py -m gpu -q -p no:cacheprovider -k "variant" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_fullsize_gpu.py -m gpu -q -p no:cacheprovider -k "1024 or sfs" 2>&1 | tail -2
