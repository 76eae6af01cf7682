timeout 300 python scripts/exp/ktime.py sfs 2>&1 | grep '^{'
timeout 300 python scripts/exp/ktime.py arap_warp 8192 2>&1 | grep '^{'
timeout 600 python bench.py --config sfs --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['avg_launch_us'], d['roofline_jtf']['avg_launch_us'])"
