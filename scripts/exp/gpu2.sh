for c in "arap_warp 8192" "poisson 8192" "arap_warp 1024" "poisson 512" "sfs 0"; do timeout 300 python scripts/exp/var_times.py $c 2>&1 | grep -v Warn; done
timeout 900 python -m pytest tests/test_golden_gpu.py -m gpu -q -p no:cacheprovider -k "variant_parity" -x 2>&1 | tail -15
