MO_B200_NOGRAPH=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ll_arap8192.csv python scripts/exp/one_solve.py arap_warp 8192 > gpurun_out/ll.log 2>&1
run() { timeout 300 env "$@" 2>&1 | grep '^{' ; }
run MO_B200_JTJ=lc python scripts/exp/ktime.py arap_warp 8192
run MO_B200_JTJ=lc MO_B200_JTJ8_MINB=7 python scripts/exp/ktime.py arap_warp 8192
run MO_B200_JTJ=lc MO_B200_JTJ8_MINB=8 python scripts/exp/ktime.py arap_warp 8192
run MO_B200_JTJ=lc MO_B200_JTJ8_NBUF=8 python scripts/exp/ktime.py arap_warp 8192
run MO_B200_JTJ=lc MO_B200_JTJ8_R=4 python scripts/exp/ktime.py arap_warp 8192
run MO_B200_JTJ=lc MO_B200_JTJ8_R=1 MO_B200_JTJ8_NBUF=8 python scripts/exp/ktime.py arap_warp 8192
