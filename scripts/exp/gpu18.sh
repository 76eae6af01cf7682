O=gpurun_out/g18; mkdir -p $O
for i in 1 2; do timeout 300 python scripts/exp/ktime.py sfs 2>&1 | grep '^{'; done
timeout 600 env MO_B200_JTJ=lct MO_B200_BM=bm8 ncu --set full --clock-control none --import-source on -k regex:mo_gather_jtj9t_0 -s 3 -c 1 -o $O/jtj9t python scripts/exp/one_apply.py arap_warp 8192 6 > $O/ncu.log 2>&1; tail -1 $O/ncu.log
