for v in "0 1" "5 1" "6 1" "5 2" "4 2"; do set -- $v; export MO_B200_JTJ2_MINB=$1 MO_B200_JTJ2_UNROLL=$2
for c in "--config arap_warp" "--config arap_warp --size 8192" "--config poisson --size 8192" "--config sfs"; do
timeout 300 python bench.py $c --steps 2 --warmup 1 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('minb=$1 unroll=$2', d['config']['workload'], round(d['value'],3), round(d['roofline']['avg_launch_us'],1), round(d['roofline']['frac'],3))"
done; done
