for c in "arap_warp 8192" "arap_warp 1024" "sfs 0" "poisson 8192"; do timeout 300 python scripts/exp/var_times.py $c 2>&1 | grep -v Warn | grep "variant [89]\|apply"; done
timeout 900 python -m pytest tests/test_golden_gpu.py -m gpu -q -p no:cacheprovider -k "variant_parity" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_fullsize_gpu.py -m gpu -q -p no:cacheprovider -k "arap_1024" 2>&1 | tail -2
