for c in "poisson 8192" "poisson 512" "arap_warp 8192"; do timeout 300 python scripts/exp/ktime.py $c 2>&1 | grep '^{'; done
timeout 300 python scripts/exp/var_times.py poisson 8192 2>&1 | grep -v Warn | tail -13
