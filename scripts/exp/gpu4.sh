run() { timeout 300 env "$@" 2>&1 | grep '^{' ; }
for c in "arap_warp 8192" "poisson 8192" "arap_warp 1024" "poisson 512"; do
  run MO_B200_JTJ=ws python scripts/exp/ktime.py $c
  run MO_B200_JTJ=lc python scripts/exp/ktime.py $c
  run MO_B200_JTJ=gather python scripts/exp/ktime.py $c
done
timeout 900 python -m pytest tests/test_golden_gpu.py -m gpu -q -p no:cacheprovider -k "variant_parity" 2>&1 | tail -5
